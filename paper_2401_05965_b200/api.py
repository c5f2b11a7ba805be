"""Reference-shaped entry points of the B200 executor.

Same names, arguments and error behaviour as the reference interpreter
(pkg/src/shardplan/interpreter.py) so a caller can switch by changing the
import.  Everything executes on the GPU through the C ABI; the single-device
evaluation that ``check_equivalence`` compares against is itself run on the
GPU (the graph's trivial one-device program in fp32), not on the host.
"""
from __future__ import annotations

import atexit
import hashlib
import json
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from .executor import ExecConfig, ExecutionError, Executor, LocalGroup, NcclGroup
from .graph_ir import Graph
from .program import DistributedProgram, Instruction
from .sharding import build_shard_table  # noqa: F401  (re-exported, interpreter.py:205)

_OP_KIND = {"MatMul": "matmul", "ElemwiseUnary": "elemwise_unary", "ElemwiseBinary": "elemwise_binary",
            "Reduce": "reduce", "Identity": "identity"}

DEFAULT_RTOL = {"bf16": 2e-2, "fp32": 1e-3}


def _as_program(program) -> DistributedProgram:
    if hasattr(program, "instrs"):
        return DistributedProgram(instrs=tuple(program.instrs), loss=program.loss)
    instrs = tuple(program)
    if not instrs:
        raise ExecutionError("cannot run an empty program")
    return DistributedProgram(instrs=instrs, loss=instrs[-1].ref)


def single_device_program(g: Graph) -> DistributedProgram:
    """The graph as a one-device program (every tensor in full form)."""
    instrs = []
    for n in g.nodes:
        if n.op in ("Placeholder", "Parameter"):
            instrs.append(Instruction(n.op.lower(), n.id, output=f"{n.id}@full"))
        else:
            instrs.append(Instruction(_OP_KIND[n.op], n.id, operands=tuple(f"{i}@full" for i in n.inputs),
                                      output=f"{n.id}@full", dims=n.dims, tag=n.tag))
    return DistributedProgram(instrs=tuple(instrs), loss=g.loss)


_GROUPS: dict = {}
_EXECUTORS: "OrderedDict" = OrderedDict()
_CACHE_SIZE = 8


def _default_group(m: int):
    """The device group of an m-device run: all m devices on this GPU, or —
    under torch.distributed with world size m — this process's rank over
    NCCL, created ONCE per process and reused by every later call."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() == m and m > 1:
        key = ("nccl", m, dist.get_rank())
        if key not in _GROUPS:
            _GROUPS[key] = NcclGroup.from_torch_distributed()
        return _GROUPS[key]
    return LocalGroup(m)


def _cache_key(prog: DistributedProgram, m: int, shard_table: dict, shapes: dict, cfg: ExecConfig, group) -> tuple:
    table = tuple(sorted((str(k[0]), int(k[1]), tuple(int(x) for x in v)) for k, v in shard_table.items()))
    # the whole instruction content (tags and dims included — canonical() omits them)
    digest = hashlib.sha256(json.dumps(prog.to_json(), sort_keys=True).encode()).hexdigest()
    return (digest, m, table, tuple(sorted(shapes.items())), repr(cfg),
            type(group).__name__, id(group) if group.distributed else m)


def compiled(prog: DistributedProgram, m: int, shard_table: dict, shapes: dict, cfg: ExecConfig,
             group=None) -> Executor:
    """The compiled executor of (program, m, shard table, source shapes,
    config, device group), built once and reused: compilation (shape
    inference, the adjoint program, launch batching, epilogue fusion, buffer
    allocation, peer-buffer registration) is paid by the first call only, so
    a repeated run costs one forward pass (LRU of the last 8)."""
    group = group or _default_group(m)
    key = _cache_key(prog, m, shard_table, shapes, cfg, group)
    ex = _EXECUTORS.get(key)
    if ex is not None:
        _EXECUTORS.move_to_end(key)
        return ex
    ex = Executor(prog, m, shard_table, shapes, group=group, config=cfg)
    _EXECUTORS[key] = ex
    while len(_EXECUTORS) > _CACHE_SIZE:
        _, old = _EXECUTORS.popitem(last=False)
        _release(old)
    return ex


def _release(ex: Executor):
    shared = ex.group.distributed   # a cached group outlives its executors
    if shared:
        ex.group, group = None, ex.group
    try:
        ex.close()
    finally:
        if shared:
            ex.group = group


def clear_cache() -> None:
    """Close every cached executor and the process's device groups."""
    while _EXECUTORS:
        _, ex = _EXECUTORS.popitem(last=False)
        _release(ex)
    for g in _GROUPS.values():
        g.close()
    _GROUPS.clear()


atexit.register(clear_cache)


def run_distributed(program, m: int, inputs: dict, shard_table: dict, debug: bool = False,
                    reference: dict | None = None, *, dtype: str = "bf16", group=None,
                    config: ExecConfig | None = None) -> list:
    """Execute a distributed program; returns the per-device loss values
    (interpreter.py:217).  With ``debug`` and ``reference`` values every
    realised distributed tensor is re-checked against its declared form
    (interpreter.py:172 check_form, at the working precision's rtol)."""
    prog = _as_program(program)
    shapes = {}
    for ins in prog.instrs:
        if ins.kind.startswith(("placeholder", "parameter")):
            if ins.ref not in inputs:
                raise ExecutionError(f"no binding for source tensor {ins.ref!r}")
            shapes[ins.ref] = tuple(np.shape(inputs[ins.ref]))
    cfg = config or ExecConfig(dtype=dtype)
    ex = compiled(prog, m, shard_table, shapes, cfg, group)
    ex.load(inputs)
    ex.forward()
    losses = ex.losses()
    if debug:
        if reference is None:
            raise AssertionError("debug mode needs reference values")
        _debug_check(ex, prog, reference, DEFAULT_RTOL.get(cfg.dtype, 2e-2))
    return [np.float64(v) for v in losses]


def _debug_check(ex: Executor, prog: DistributedProgram, reference: dict, rtol: float):
    """interpreter.py:172 check_form for every instruction's output: the m
    device instances — gathered from every rank when one process runs one
    device — must realise the declared property of the reference value: Id =
    every replica equal to the reference, AG(d) = the concatenation along d,
    AR = the sum; guard properties raise, as in the reference."""
    from .program import ALL_GATHER, ALL_REDUCE, IDENTITY, form_of_dist_id

    for ins in prog.instrs:
        prop = form_of_dist_id(ins.output)
        mine = {r: ex.tensor(ins.output, r).float().cpu().numpy().astype(np.float64) for r in ex.group.local_ranks}
        if ex.group.distributed:
            insts = ex.group.exchange(mine[ex.group.rank])
        else:
            insts = [mine[r] for r in range(ex.m)]
        want = np.asarray(reference[prop.ref], dtype=np.float64)
        scale = np.maximum(np.abs(want), 1.0)

        def close(got):
            return got.shape == want.shape and bool(np.all(np.abs(got - want) <= rtol * scale))

        if prop.kind == IDENTITY:
            ok = all(close(inst) for inst in insts)
        elif prop.kind == ALL_GATHER:
            ok = close(np.concatenate(insts, axis=prop.axis))
        elif prop.kind == ALL_REDUCE:
            ok = close(sum(insts[1:], insts[0]))
        else:
            raise ValueError(f"cannot check guard property {prop}")
        if not ok:
            raise ExecutionError(f"{ins.canonical()} violates its declared property {prop}")


def run_single(g: Graph, inputs: dict, *, dtype: str = "fp32") -> np.float64:
    """Single-device loss (interpreter.py:62), evaluated on the GPU."""
    for n in g.nodes:
        if n.op in ("Placeholder", "Parameter"):
            if n.id not in inputs:
                raise ExecutionError(f"no binding for source tensor {n.id!r}")
            if tuple(np.shape(inputs[n.id])) != n.shape:
                raise ExecutionError(f"binding for {n.id!r} has shape {np.shape(inputs[n.id])}, want {n.shape}")
    return run_distributed(single_device_program(g), 1, inputs, {}, dtype=dtype)[0]


def random_inputs(g: Graph, rng: np.random.Generator, integer: bool = False) -> dict:
    """Seeded source bindings, identical draws to interpreter.py:252."""
    out = {}
    for n in g.nodes:
        if n.op in ("Placeholder", "Parameter"):
            if integer:
                out[n.id] = rng.integers(-4, 5, size=n.shape).astype(np.float64)
            else:
                out[n.id] = rng.standard_normal(n.shape)
    return out


@dataclass(frozen=True)
class EquivalenceReport:
    trials: int
    max_rel_err: float
    passed: bool


def check_equivalence(g: Graph, program, m: int, shard_table: dict, trials: int = 5, seed: int = 0,
                      rtol: float | None = None, *, dtype: str = "bf16") -> EquivalenceReport:
    """interpreter.py:264 — every device's loss against the single-device loss
    over seeded random inputs; the tolerance defaults to the working
    precision's (2e-2 bf16, 1e-3 fp32) instead of the float64 reference's 1e-9."""
    rtol = DEFAULT_RTOL[dtype] if rtol is None else rtol
    worst = 0.0
    for t in range(trials):
        inputs = random_inputs(g, np.random.default_rng(seed + t))
        expected = float(run_single(g, inputs))
        losses = run_distributed(program, m, inputs, shard_table, dtype=dtype)
        scale = max(abs(expected), 1.0)
        for v in losses:
            worst = max(worst, abs(float(v) - expected) / scale)
    return EquivalenceReport(trials=trials, max_rel_err=worst, passed=worst <= rtol)
