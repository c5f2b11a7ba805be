"""B200 executor for HAP-synthesized distributed programs.

Drop-in for the reference interpreter's run path (pkg/src/shardplan/
interpreter.py: ``run_distributed`` :217, ``execute_instruction`` :118,
``check_equivalence`` :264): it takes the same program, device count and
shard table, but every instruction runs as hand-written sm_100a CUDA through
the C ABI (include/hap_b200.h) — tcgen05 GEMMs, vectorised elementwise and
reduction kernels, NCCL collectives over NVLink — and it also runs the
training step the reference cannot: the adjoint program (backward), the
parameter-gradient synchronisation (all-reduce or sufficient-factor
broadcasting, chosen by the cost model) and an SGD update.

Device groups:
  * ``NcclGroup`` — one process per GPU, rank j executes device j of the
    program; collectives are NCCL calls on the compute stream.
  * ``LocalGroup`` — all m program devices on one GPU in lock step, the
    reference interpreter's own execution model; collectives become local
    copy / sum kernels.  Used for parity tests of m-device programs on a
    single GPU.

The compile step turns the program into a flat list of C-ABI launches with
every pointer and size resolved, so a step is a loop of ctypes calls — or a
single CUDA-graph replay.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import BF16, F32, check
from .program import (ALL_GATHER, ALL_REDUCE, IDENTITY, DistributedProgram, Instruction,
                      form_of_dist_id)
from .sharding import offsets

SOURCE_KINDS = ("placeholder", "placeholder_shard", "parameter", "parameter_shard")
_TORCH = {F32: torch.float32, BF16: torch.bfloat16}


class ExecutionError(RuntimeError):
    """A program that cannot execute (unsound plan, missing binding or shard
    sizes) — same contract as the reference's interpreter.ExecutionError."""


# ---------------------------------------------------------------------------- buffers

@dataclass
class Buf:
    tensor: torch.Tensor
    dtype: int
    shape: tuple

    @property
    def ptr(self) -> int:
        return self.tensor.data_ptr()

    @property
    def numel(self) -> int:
        return int(math.prod(self.shape))


def _view(shape: tuple, axis: int) -> tuple[int, int, int]:
    """(outer, extent, inner) of ``shape`` around ``axis``."""
    return (int(math.prod(shape[:axis])), int(shape[axis]), int(math.prod(shape[axis + 1:])))


# ---------------------------------------------------------------------------- groups

class LocalGroup:
    """All m program devices emulated on the current GPU (lock step)."""

    distributed = False

    def __init__(self, m: int):
        self.m = m
        self.rank = 0
        self.local_ranks = list(range(m))
        self.comm = None
        self.comm_grad = None

    def close(self):
        pass


def _dist_exchange(obj) -> list:
    import torch.distributed as dist

    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


class NcclGroup:
    """One program device per process; collectives over NCCL (C ABI) or the
    hand-written NVLink kernels, whichever the cost model picks per call site.

    Two communicators: ``comm`` carries the program's collectives on the
    compute stream, ``comm_grad`` the parameter-gradient all-reduces on a side
    stream that overlaps the rest of the backward pass (NCCL operations on
    one communicator must not run concurrently from two streams)."""

    distributed = True
    in_process = False

    def __init__(self, rank: int, m: int, comm_handle, grad_handle=None):
        self.m = m
        self.rank = rank
        self.local_ranks = [rank]
        self.comm = comm_handle
        self.comm_grad = grad_handle

    @staticmethod
    def _init_comm(rank: int, world: int):
        import torch.distributed as dist

        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            check(_lib.lib().hap_comm_unique_id(uid), "hap_comm_unique_id")
        obj = [bytes(uid.raw) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        handle = ctypes.c_void_p()
        check(_lib.lib().hap_comm_init(ctypes.byref(handle), obj[0], world, rank), "hap_comm_init")
        return handle

    @classmethod
    def from_torch_distributed(cls) -> "NcclGroup":
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        return cls(rank, world, cls._init_comm(rank, world), cls._init_comm(rank, world))

    def exchange(self, obj) -> list:
        """Every rank's ``obj``, rank-ordered (host-side, compile time only)."""
        return _dist_exchange(obj)

    def close(self):
        for name in ("comm", "comm_grad"):
            handle = getattr(self, name)
            if handle is not None:
                check(_lib.lib().hap_comm_destroy(handle), "hap_comm_destroy")
                setattr(self, name, None)


class PeerGroup:
    """One program device per executor whose collectives are ONLY the
    hand-written NVLink peer-memory kernels (p2p.cu: push all-gather, direct
    reduce-scatter, two-shot all-reduce, push all-to-all) — no NCCL.

    Two forms: one process per GPU (``from_torch_distributed``: buffers are
    exchanged as CUDA IPC handles over any torch.distributed backend), or all
    ranks inside ONE process (``thread_peer_groups``: each rank an Executor on
    its own stream, built and stepped in its own thread, buffers exchanged as
    plain device pointers — ``hap_symm_open_local``).  The in-process form
    runs the multi-device path on a single GPU, ranks side by side under SM
    caps, which is how the 1-GPU test box verifies it."""

    distributed = True
    comm = None
    comm_grad = None

    def __init__(self, rank: int, m: int, exchange=None):
        self.m = m
        self.rank = rank
        self.local_ranks = [rank]
        self._exchange = exchange
        self.in_process = exchange is not None

    @classmethod
    def from_torch_distributed(cls) -> "PeerGroup":
        import torch.distributed as dist

        return cls(dist.get_rank(), dist.get_world_size())

    def exchange(self, obj) -> list:
        if self._exchange is not None:
            return self._exchange(self.rank, obj)
        return _dist_exchange(obj)

    def close(self):
        pass


def thread_peer_groups(m: int, timeout: float = 120.0) -> list:
    """m PeerGroups of one process whose exchange is an in-process rendezvous
    (a barrier across the m threads that build the m executors)."""
    import threading

    barrier = threading.Barrier(m, timeout=timeout)
    slots: list = [None] * m

    def exchange(rank: int, obj):
        slots[rank] = obj
        barrier.wait()
        out = list(slots)
        barrier.wait()
        return out

    return [PeerGroup(r, m, exchange=exchange) for r in range(m)]


def run_ranks(fns: list) -> list:
    """Run fns[r]() for every rank in its own thread (ctypes calls release the
    GIL, so the ranks enqueue concurrently and a rank's peer-memory kernel
    never waits on a host thread that is blocked behind it); re-raises the
    first failure."""
    import threading

    out: list = [None] * len(fns)
    err: list = []

    def body(r):
        try:
            out[r] = fns[r]()
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            err.append(exc)

    threads = [threading.Thread(target=body, args=(r,)) for r in range(len(fns))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if err:
        raise err[0]
    return out


_CUDART = None


def _cudart():
    """The CUDA runtime library the process already uses (PyTorch's)."""
    global _CUDART
    if _CUDART is None:
        import glob

        base = os.path.dirname(torch.__file__)
        cands = sorted(glob.glob(os.path.join(base, "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*")) +
                       glob.glob(os.path.join(base, "lib", "libcudart*.so*")))
        if not cands:
            raise ExecutionError("libcudart not found next to torch")
        _CUDART = ctypes.CDLL(cands[0])
    return _CUDART


_FREE_STREAMS: dict = {}   # device index -> streams no live executor holds


def _acquire_stream(dev: int) -> int:
    free = _FREE_STREAMS.setdefault(dev, [])
    if free:
        return free.pop()
    ptr = ctypes.c_void_p()
    with torch.cuda.device(dev):
        rc = _cudart().cudaStreamCreateWithFlags(ctypes.byref(ptr), 1)   # cudaStreamNonBlocking
    if rc:
        raise ExecutionError(f"cudaStreamCreateWithFlags failed ({rc})")
    return ptr.value


def _release_streams(dev: int, ptrs: list) -> None:
    while ptrs:
        _FREE_STREAMS.setdefault(dev, []).append(ptrs.pop())


class _HostStream:
    """Stand-in for a CUDA stream when the executor only COMPILES on the host
    (device "cpu": the dry-run form used by the CPU tests to check the
    per-rank collective planning without a GPU).  Never runs a kernel."""

    cuda_stream = 0

    def synchronize(self):
        pass

    def wait_event(self, _event):
        pass


class _HostEvent:
    def record(self, _stream=None):
        pass


# ---------------------------------------------------------------------------- config

@dataclass
class ExecConfig:
    dtype: str = "bf16"               # working precision of activations ("bf16" | "fp32")
    sm_caps: list | None = None       # per program-device SM cap (heterogeneity emulation)
    lr: float = 0.0                   # SGD learning rate of train_step
    grad_sync: str = "auto"           # "auto" (cost model) | "all_reduce" | "sfb"
    gather: str = "auto"              # all_gather / reduce_scatter impl: "auto" = "kernel" (NVLink
                                      # peer-memory kernel) | "padded" (NCCL, max-shard padding) |
                                      # "sendrecv" (NCCL grouped point-to-point)
    p2p_push: bool = os.environ.get("HAP_P2P_PUSH", "1") == "1"   # "kernel" collectives on registered
                                      # buffers: all-gathers store straight into every rank's output (NVLink
                                      # writes), reduce-scatters read the peers' partials in place; no staging
                                      # (else: staged pull kernels)
    input_grads: bool = False         # also differentiate w.r.t. placeholders
    cluster: object = None            # ClusterSpec for the cost-model choices
    ratios: tuple | None = None       # ratio row the plan was made with (cost model)
    batch_gemms: bool = True          # merge runs of matmuls into batched launches
    fuse_elementwise: bool = True     # fuse swish / gate elementwise chains
    fuse_epilogue: bool = True        # fold elementwise work into the producing GEMM's epilogue (bf16
                                      # outputs): residual adds, deferred gradient copies, the swish
                                      # adjoint after the dz GEMM
    fuse_swish_fwd: bool = os.environ.get("HAP_FUSE_SWISH_FWD", "1") == "1"   # also y = f(x), z = x*y
                                      # after the x GEMM (three outputs per tile)
    overlap_sfb: bool = True          # NCCL groups: SFB factor gathers on a side stream (activations
                                      # during the forward), weight-gradient GEMMs at the end of backward
    bucket_bytes: int = 32 << 20      # NCCL groups: gradients all-reduced in buckets of about this size
    autotune: str = os.environ.get("HAP_AUTOTUNE", "table")   # GEMM tile shape / split-K per launch
                                      # signature: "table" = the committed B200 table (_lib.TUNE_TABLE), the
                                      # host heuristic for signatures it lacks — the same choice, hence the
                                      # same rounding, in every process; "time" = also time the signatures
                                      # the table lacks (hap_matmul_tune, fastest kept); "off" = heuristic
    wgrad_stream: bool = os.environ.get("HAP_WGRAD_STREAM", "0") == "1"   # parameter-gradient GEMMs on a
                                      # side stream, to run in the tails of the activation-gradient chain;
                                      # off: measured no gain (persistent GEMMs keep their static tile
                                      # schedule, so a late-starting launch only stretches the chain)
    sgd_overlap: str = os.environ.get("HAP_SGD_OVERLAP", "auto")   # "1": update each parameter group on
                                      # a side stream as soon as the backward no longer touches it (its
                                      # gradient final, its weights read for the last time), so the
                                      # HBM-bound update runs beside the remaining backward GEMMs; "auto":
                                      # only when the update is long against the backward GEMMs (few
                                      # tokens per parameter: MoE +4 %, BERT -0.5 % measured)


@dataclass
class Op:
    fn: object
    args: tuple
    what: str
    kernel: bool = True               # launches one of our kernels (vs NCCL / memcpy)
    gemm: dict | None = None          # matmul record (for launch batching)
    meta: dict | None = None          # peer-memory collectives: what the launch moves (buffers, sizes)


# ---------------------------------------------------------------------------- executor

def price_grad_sync(spec, ratios, weight: str, kdim: int, ndim: int, uses, shared: dict | None = None) -> str:
    """HAP's SFB rule for one replicated [kdim, ndim] weight whose uses are
    row-sharded matmuls ``(x_ref, y_ref, rows)``: all-reduce the partial dW
    (plus the ratio-sharded dW GEMMs) against all-gathering x and dy and
    rebuilding dW at full batch on every device — each priced with the
    reference cost model's collective times (cost_model.comm_time) and the
    slowest device's GEMM time.  ``shared`` maps a factor to the number of
    weights whose SFB reuses its one gather (the executor gathers a factor
    once per source buffer: both experts of a layer read the same input), so
    each weight is charged its share.  Returns "sfb" or "all_reduce"."""
    from .cost_model import ClusterSpec, comm_time

    if not isinstance(spec, ClusterSpec):
        spec = ClusterSpec.from_dict(spec)
    row = tuple(ratios) if ratios else tuple(d.flops_per_second / spec.total_rate for d in spec.devices)
    rates = [d.flops_per_second for d in spec.devices]
    t_ar = comm_time(Instruction("all_reduce", weight, elements=kdim * ndim), row, spec)
    t_sfb = 0.0
    for x_ref, y_ref, rows in uses:
        flops = 2 * rows * kdim * ndim
        t_sfb += comm_time(Instruction("all_gather", x_ref, elements=rows * kdim), row, spec) / \
            max(1, (shared or {}).get(x_ref, 1))
        t_sfb += comm_time(Instruction("all_gather", y_ref, elements=rows * ndim), row, spec)
        # SFB replicates the weight-gradient GEMM at full batch on every device;
        # all-reduce keeps it sharded.
        t_sfb += max(flops / rt for rt in rates)
        t_ar += max(flops * b / rt for b, rt in zip(row, rates))
    return "sfb" if t_sfb < t_ar else "all_reduce"


class Executor:
    """Compiled executor of one distributed program on this process's devices."""

    def __init__(self, program: DistributedProgram, m: int, shard_table: dict,
                 source_shapes: dict, group=None, config: ExecConfig | None = None,
                 device: torch.device | None = None):
        self.lib = _lib.lib()
        self.program = program
        self.m = m
        self.table = {(k[0], int(k[1])): list(v) for k, v in shard_table.items()}
        self.source_shapes = {k: tuple(v) for k, v in source_shapes.items()}
        self.group = group or LocalGroup(m)
        if self.group.m != m:
            raise ExecutionError(f"device group has {self.group.m} devices, program needs {m}")
        self.cfg = config or ExecConfig()
        self.wdt = BF16 if self.cfg.dtype == "bf16" else F32
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        # device "cpu": compile only (the op list, buffers on the host) — the
        # CPU tests' dry run of the per-rank planning; nothing can be launched
        self.dry = self.device.type == "cpu"
        self.stream = self._stream()
        self.caps = list(self.cfg.sm_caps) if self.cfg.sm_caps else [0] * m
        self.ops_fwd: list[Op] = []
        self.ops_bwd: list[Op] = []
        self._ops = self.ops_fwd
        self.bufs: dict[tuple[str, int], Buf] = {}
        self.grads: dict[tuple[str, int], Buf] = {}
        self.masters: dict[tuple[str, int], Buf] = {}
        self.shapes: dict[str, list[tuple]] = {}
        self.dtypes: dict[str, int] = {}
        self.sync_choice: dict[str, str] = {}
        self.graph: torch.cuda.CUDAGraph | None = None
        self._pool: list[Buf] = []
        self.sfb: dict = {}
        self.sfb_done: set = set()
        self.overlapped: set = set()
        self._grad_ready_at: dict = {}
        self.comm_stream = None
        self.aliased: set = set()
        self._n_contrib: dict = {}
        self.bytes_allocated = 0
        self.source_dids = {i.output for i in program.instrs if i.kind in SOURCE_KINDS}
        self._check_program()
        self._infer()
        self._allocate()
        self._symm: dict = {}            # stream tag -> peer-memory context
        self._p2p_bytes: dict = {}       # stream tag -> largest staging need
        self._p2p_regs: list = []        # (stream tag, registered Buf, slot): push all-gather outputs,
                                         # direct reduce-scatter partials
        self._emit_on = None             # stream the next ops are emitted on (None: self.stream)
        self.impl_choice: list = []      # (kind, bytes, "p2p" | "nccl", priced p2p s, priced nccl s) per call site
        self._sfb_full: dict = {}        # gathered SFB factors, keyed by source buffer
        self._sfb_pending: list = []     # deferred SFB weight-gradient GEMMs
        self._sgd_items: dict = {}       # (rank, weight dtype) -> [(master, grad, weight)] (_compile_sgd)
        self._plan_sfb()
        self._compile_forward()
        self._compile_backward()
        if self.cfg.batch_gemms:
            self.ops_fwd[:] = self._batch_gemms(self.ops_fwd)
            self.ops_bwd[:] = self._batch_gemms(self.ops_bwd)
        self.wgrad_stats = (0, 0, 0)
        if self.cfg.wgrad_stream:
            self.ops_bwd[:] = self._offload_wgrad(self.ops_bwd)
        self.sgd_stats = (0, 0)
        if self.cfg.lr and self._sgd_items and self._want_sgd_overlap():
            self._overlap_sgd()
        self.tuned_signatures = 0
        if self.wdt == BF16 and not self.dry:
            self._autotune()
        self._create_symm()
        if not self.dry:
            # compile-time initialisation (zeroed gradient buckets, tuning
            # launches) ran on torch's streams, which the executor's own
            # non-blocking stream does not wait for
            torch.cuda.synchronize(self.device)

    def _stream(self):
        """A CUDA stream no other live executor uses (non-blocking): torch's
        torch.cuda.Stream() hands out streams round-robin from a pool of 32 per
        device, so two executors of one process — the in-process ranks of
        thread_peer_groups — could be given the same cudaStream_t, and a rank's
        peer kernel spinning for its partner would then sit in front of that
        partner's work.  Streams come from a process-wide free list, go back to
        it when the executor is closed or collected, and are never destroyed
        (torch may still record events on them for tensors they touched)."""
        if self.dry:
            return _HostStream()
        dev = self.device.index if self.device.index is not None else torch.cuda.current_device()
        if "_own_streams" not in self.__dict__:
            import weakref

            self._own_streams = []
            weakref.finalize(self, _release_streams, dev, self._own_streams)
        ptr = _acquire_stream(dev)
        self._own_streams.append(ptr)
        return torch.cuda.ExternalStream(ptr, device=self.device)

    def _event(self):
        return _HostEvent() if self.dry else torch.cuda.Event()

    def _autotune(self):
        """Tile shapes of the GEMM launches.  "table" / "time": import the
        committed tuning table; "time" additionally runs one hap_matmul_tune
        per distinct launch signature the table lacks (layers repeat shapes):
        the library times every tile shape / split of the batch on scratch
        outputs and uses the fastest from then on."""
        mode = {True: "time", False: "off", "1": "time", "0": "off"}.get(self.cfg.autotune, self.cfg.autotune)
        if mode == "off":
            return
        _lib.load_tune_table()
        if mode != "time":
            return
        seen = set()
        for op in self.ops_fwd + self.ops_bwd:
            if op.gemm is None:
                continue
            descs, count, sum_k, in_dt, out_dt, cap, stream = op.args
            key = (count, sum_k, in_dt, out_dt, cap) + tuple(
                (d.M, d.N, d.K, d.transA, d.transB, d.epi, d.accumulate, d.lda, d.ldb, d.ldc)
                for d in descs[:count])
            if key in seen:
                continue
            seen.add(key)
            check(self.lib.hap_matmul_tune(descs, count, sum_k, in_dt, out_dt, cap, stream), "hap_matmul_tune")
        torch.cuda.synchronize(self.device)
        self.tuned_signatures = len(seen)

    # ------------------------------------------------------------------ analysis
    def _sizes(self, ref: str, axis: int) -> list[int]:
        try:
            sizes = self.table[(ref, axis)]
        except KeyError:
            raise ExecutionError(f"shard table lacks sizes for tensor {ref!r} axis {axis}") from None
        if len(sizes) != self.m:
            raise ExecutionError(f"shard table entry for {ref!r} axis {axis} has {len(sizes)} "
                                 f"entries for {self.m} devices")
        return sizes

    def _check_program(self):
        if not self.program.instrs:
            raise ExecutionError("cannot run an empty program")
        seen = set()
        for ins in self.program.instrs:
            for d in ins.operands:
                if d not in seen:
                    raise ExecutionError(f"instruction {ins.canonical()} reads unrealized tensor {d!r}")
            if ins.kind in SOURCE_KINDS and ins.ref not in self.source_shapes:
                raise ExecutionError(f"no binding for source tensor {ins.ref!r}")
            seen.add(ins.output)

    def _infer(self):
        """Per-device shapes and dtypes of every distributed tensor."""
        m = self.m
        for ins in self.program.instrs:
            k = ins.kind
            ops = [self.shapes[d] for d in ins.operands]
            dts = [self.dtypes[d] for d in ins.operands]
            if k in ("placeholder", "parameter"):
                full = self.source_shapes[ins.ref]
                out = [full] * m
                dt = self.wdt
            elif k in ("placeholder_shard", "parameter_shard"):
                full = self.source_shapes[ins.ref]
                if not 0 <= ins.axis < len(full):
                    raise ExecutionError(f"shape mismatch executing {ins.canonical()}: axis {ins.axis}")
                sizes = self._sizes(ins.ref, ins.axis)
                if sum(sizes) != full[ins.axis]:
                    raise ExecutionError(f"shard sizes {sizes} do not cover extent {full[ins.axis]}")
                out = [tuple(s if a == ins.axis else e for a, e in enumerate(full)) for s in sizes]
                dt = self.wdt
            elif k == "matmul":
                out = []
                for a, b in zip(*ops):
                    if len(a) != 2 or len(b) != 2 or a[1] != b[0]:
                        raise ExecutionError(f"shape mismatch executing {ins.canonical()}: {a} x {b}")
                    out.append((a[0], b[1]))
                dt = self.wdt
            elif k in ("elemwise_unary", "identity"):
                out = list(ops[0])
                dt = dts[0]
            elif k == "elemwise_binary":
                for a, b in zip(*ops):
                    if a != b:
                        raise ExecutionError(f"shape mismatch executing {ins.canonical()}: {a} vs {b}")
                out = list(ops[0])
                dt = F32 if F32 in dts else self.wdt
            elif k == "reduce":
                out = [tuple(e for a, e in enumerate(s) if a not in ins.dims) for s in ops[0]]
                dt = F32
            elif k == "all_reduce":
                if len(set(ops[0])) != 1:
                    raise ExecutionError(f"shape mismatch executing {ins.canonical()}")
                out = list(ops[0])
                dt = dts[0]
            elif k in ("all_gather", "grouped_broadcast"):
                s0 = ops[0][0]
                ext = sum(s[ins.axis] for s in ops[0])
                out = [tuple(ext if a == ins.axis else e for a, e in enumerate(s0))] * m
                dt = dts[0]
            elif k == "reduce_scatter":
                sizes = self._sizes(ins.ref, ins.axis)
                s0 = ops[0][0]
                if sum(sizes) != s0[ins.axis]:
                    raise ExecutionError(f"shard sizes {sizes} do not cover extent {s0[ins.axis]}")
                out = [tuple(sz if a == ins.axis else e for a, e in enumerate(s0)) for sz in sizes]
                dt = dts[0]
            elif k == "all_to_all":
                sizes = self._sizes(ins.ref, ins.axis2)
                s0 = ops[0][0]
                ext1 = sum(s[ins.axis] for s in ops[0])
                if sum(sizes) != s0[ins.axis2]:
                    raise ExecutionError(f"shard sizes {sizes} do not cover extent {s0[ins.axis2]}")
                out = [tuple(ext1 if a == ins.axis else (sz if a == ins.axis2 else e)
                             for a, e in enumerate(s0)) for sz in sizes]
                dt = dts[0]
            else:
                raise ExecutionError(f"unsupported instruction kind {k!r}")
            self.shapes[ins.output] = out
            self.dtypes[ins.output] = dt
        # Which tensors need gradients: anything downstream of a parameter
        # (and of placeholders when input gradients are requested).
        self.req: dict[str, bool] = {}
        for ins in self.program.instrs:
            if ins.kind in SOURCE_KINDS:
                self.req[ins.output] = ins.kind.startswith("parameter") or self.cfg.input_grads
            else:
                self.req[ins.output] = any(self.req[d] for d in ins.operands)

    def _new(self, shape, dtype) -> Buf:
        """Device buffer that lives as long as the executor: compiled ops hold
        raw pointers, so every buffer (temporaries included) is pinned here."""
        t = torch.empty(max(1, int(math.prod(shape))), dtype=_TORCH[dtype], device=self.device)
        buf = Buf(t, dtype, tuple(shape))
        self._pool.append(buf)
        self.bytes_allocated += t.numel() * t.element_size()
        return buf

    def _allocate(self):
        for did, shapes in self.shapes.items():
            for r in self.group.local_ranks:
                self.bufs[(did, r)] = self._new(shapes[r], self.dtypes[did])
        for ins in self.program.instrs:
            if ins.kind.startswith("parameter"):
                for r in self.group.local_ranks:
                    self.masters[(ins.output, r)] = self._new(self.shapes[ins.output][r], F32)
        self.loss_buf = {r: self._new((), F32) for r in self.group.local_ranks}

    # ------------------------------------------------------------------ emission
    def _emit(self, name: str, *args, kernel: bool = True, what: str = ""):
        fn = getattr(self.lib, name)
        self._ops.append(Op(fn, args, what or name, kernel))

    def _sptr(self):
        return (self._emit_on or self.stream).cuda_stream

    def _comm(self):
        """NCCL communicator of the stream being emitted on: collectives on
        the side stream use their own communicator, so the two streams never
        interleave operations on one communicator."""
        g = self.group
        return g.comm_grad if self._emit_on is not None and self._emit_on is self.comm_stream else g.comm

    def _side(self):
        if self.comm_stream is None:
            self.comm_stream = self._stream()
        return self.comm_stream

    def _copy(self, src: Buf, dst: Buf, cap: int, accumulate: int = 0, alpha: float = 1.0):
        n = src.numel if src.shape else 1
        if dst.numel != n and dst.shape:
            raise ExecutionError(f"copy of {src.shape} into {dst.shape}")
        self._emit("hap_axpy", alpha, src.ptr, src.dtype, dst.ptr, dst.dtype, n, accumulate, cap,
                   self._sptr())

    def _block(self, src: Buf, src_view, src_off, dst: Buf, dst_view, dst_off, count, cap,
               accumulate=0):
        so, se, si = src_view
        do, de, di = dst_view
        if so != do or si != di:
            raise ExecutionError(f"block copy views disagree: {src_view} vs {dst_view}")
        self._emit("hap_copy_block", src.ptr, src.dtype, se, src_off, dst.ptr, dst.dtype, de, dst_off,
                   so, count, si, accumulate, cap, self._sptr())

    def _as(self, buf: Buf, dtype: int, cap: int) -> Buf:
        """Buffer holding ``buf`` in ``dtype`` (a conversion op when needed)."""
        if buf.dtype == dtype:
            return buf
        out = self._new(buf.shape, dtype)
        self._copy(buf, out, cap)
        return out

    def _gemm(self, a: Buf, trans_a: bool, b: Buf, trans_b: bool, c: Buf, cap: int, accumulate: int,
              addend: Buf | None = None):
        """C (+)= op(A).op(B) as one hap_matmul_batch launch of a single
        descriptor (later passes may merge descriptors into batches or fold
        elementwise work into the descriptor's epilogue).  ``addend``: C =
        A.B + addend (a deferred gradient copy, see _compile_backward)."""
        am, ak = (a.shape[1], a.shape[0]) if trans_a else a.shape
        bk, bn = (b.shape[1], b.shape[0]) if trans_b else b.shape
        if ak != bk or tuple(c.shape) != (am, bn):
            raise ExecutionError(f"gemm shape mismatch {a.shape}{'T' if trans_a else ''} x "
                                 f"{b.shape}{'T' if trans_b else ''} -> {c.shape}")
        in_dt = BF16 if (a.dtype == BF16 and b.dtype == BF16) else F32
        a = self._as(a, in_dt, cap)
        b = self._as(b, in_dt, cap)
        c_out = None
        if in_dt == BF16 and (self._misaligned(a) or self._misaligned(b) or self._misaligned(c)):
            # uneven shards of a bf16 dimension (e.g. the ViT-MoE expert slices
            # 1804 / 1268 of 3072 columns) leave rows that are not 16-byte
            # pitched, which TMA cannot describe: stage misaligned operands
            # into padded copies and compute a misaligned C into a padded
            # buffer copied back, so the GEMM stays on the tcgen05 path
            if self._misaligned(a):
                a = self._pitched(a, True, cap)
            if self._misaligned(b):
                b = self._pitched(b, True, cap)
            if self._misaligned(c):
                rows, cols = c.shape
                c_out, c = c, self._pitched(c, bool(accumulate), cap)
                if addend is not None:   # C = A.B + addend: stage the addend and accumulate onto it
                    self._block(addend, (rows, cols, 1), 0, c, (rows, c.shape[1], 1), 0, cols, cap)
                    accumulate, addend = 1, None
        g = dict(A=a.ptr, lda=a.shape[1], transA=int(trans_a), B=b.ptr, ldb=b.shape[1],
                 transB=int(trans_b), C=c.ptr, ldc=c.shape[1], M=am, N=bn, K=ak,
                 accumulate=accumulate, in_dt=in_dt, out_dt=c.dtype, cap=cap,
                 stream=self._sptr(), epi=_lib.EPI_NONE, epi_tag=0, R=None, ldr=0, R2=None, ldr2=0,
                 Y=None, ldy=0, Z=None, ldz=0)
        if addend is not None:
            g.update(epi=_lib.EPI_ADD, R=addend.ptr, ldr=addend.shape[1], accumulate=0)
        desc = (_lib.GemmDesc * 1)()
        self._ops.append(Op(self.lib.hap_matmul_batch, (desc, 1, 0, in_dt, c.dtype, cap, self._sptr()),
                            "hap_matmul", True, g))
        self._sync_desc(self._ops[-1])
        if c_out is not None:
            rows, cols = c_out.shape
            self._block(c, (rows, c.shape[1], 1), 0, c_out, (rows, cols, 1), 0, cols, cap)

    @staticmethod
    def _misaligned(buf: Buf) -> bool:
        """Rows not 16-byte pitched: TMA cannot describe the matrix, and the
        GEMM would fall back to the CUDA-core kernel."""
        return len(buf.shape) == 2 and (buf.shape[1] * (2 if buf.dtype == BF16 else 4)) % 16 != 0

    def _pitched(self, buf: Buf, copy_in: bool, cap: int) -> Buf:
        """A copy of ``buf`` with its rows padded to a 16-byte pitch (the pad
        columns are never read: the GEMM's extents are the logical ones)."""
        rows, cols = buf.shape
        per = 8 if buf.dtype == BF16 else 4
        pad = self._new((rows, -(-cols // per) * per), buf.dtype)
        if copy_in:
            self._block(buf, (rows, cols, 1), 0, pad, (rows, pad.shape[1], 1), 0, cols, cap)
        return pad

    @staticmethod
    def _fill_desc(d, g: dict):
        for k in ("A", "lda", "transA", "B", "ldb", "transB", "C", "ldc", "M", "N", "K", "accumulate", "epi",
                  "epi_tag", "R", "ldr", "R2", "ldr2", "Y", "ldy", "Z", "ldz"):
            setattr(d, k, g[k])

    def _sync_desc(self, op: Op):
        """Write a single-GEMM op's record into its launch descriptor."""
        self._fill_desc(op.args[0][0], op.gemm)

    def _gemm_fusable(self, g: dict) -> bool:
        """The GEMM can take a fused epilogue: tcgen05 path, bf16 output,
        16-byte pitched buffers, one plain descriptor."""
        if not self.cfg.fuse_epilogue or g is None or g.get("members") or g["out_dt"] != BF16:
            return False
        if g["epi"] != _lib.EPI_NONE or g["ldc"] % 8 or g["C"] % 16:
            return False
        return self.lib.hap_matmul_engine(g["A"], g["lda"], g["transA"], g["B"], g["ldb"], g["transB"], g["M"],
                                          g["N"], g["K"], g["in_dt"]) == _lib.GEMM_TCGEN05

    def _producer_gemm(self, ptr: int, window: int = 8):
        """The recent single-GEMM op that wrote ``ptr`` (its C), if only GEMMs
        that do not read ``ptr`` (and stream events) were emitted after it."""
        for op in reversed(self._ops[-window:]):
            g = op.gemm
            if g is None:
                if op.what in ("event.record", "stream.wait_event"):
                    continue
                return None
            if g["C"] == ptr and not g.get("members"):
                return op
            if ptr in (g["A"], g["B"], g["R"], g["R2"], g["C"], g["Y"], g["Z"]):
                return None
        return None

    @staticmethod
    def _fusable_buf(*bufs) -> bool:
        shape = tuple(bufs[0].shape)
        return all(b.dtype == BF16 and len(b.shape) == 2 and tuple(b.shape) == shape and b.shape[1] % 8 == 0
                   and b.ptr % 16 == 0 for b in bufs)

    # ------------------------------------------------------------------ collectives
    # Every collective maps per-device source buffers to per-device outputs with
    # the reference's semantics (interpreter.py:69-101) and an `accumulate`
    # flag so adjoints can add into gradient buffers.

    def _coll_all_reduce(self, src: dict, dst: dict, accumulate: int):
        g = self.group
        if isinstance(g, LocalGroup):
            tmp = self._new(src[0].shape, src[0].dtype if src[0].dtype == F32 else F32)
            for j in range(self.m):
                self._copy(src[j], tmp, self.caps[j], accumulate=int(j > 0))
            for j in range(self.m):
                self._copy(tmp, dst[j], self.caps[j], accumulate=accumulate)
            return
        r = g.rank
        s = src[r]
        target = dst[r] if (not accumulate and dst[r].dtype == s.dtype) else self._new(s.shape, s.dtype)
        n = s.numel if s.shape else 1
        if self._use_p2p("all_reduce", n, 2 if s.dtype == BF16 else 4):
            self._p2p_all_reduce(s, target, n)
        else:
            self._emit("hap_all_reduce", self._comm(), s.ptr, target.ptr, n, s.dtype, self._sptr(), kernel=False)
        if target is not dst[r]:
            self._copy(target, dst[r], self.caps[r], accumulate=accumulate)

    def _coll_all_gather(self, src: dict, src_shapes: list, dst: dict, axis: int, accumulate: int,
                         kind: str):
        """Shards along ``axis`` (all devices' shapes ``src_shapes``) -> full
        tensor on every device."""
        g = self.group
        sizes = [s[axis] for s in src_shapes]
        offs = offsets(sizes)
        full_shape = dst[g.local_ranks[0]].shape
        if isinstance(g, LocalGroup):
            for j in range(self.m):
                for k in range(self.m):
                    self._block(src[k], _view(src[k].shape, axis), 0, dst[j], _view(full_shape, axis),
                                offs[k], sizes[k], self.caps[j], accumulate)
            return
        r = g.rank
        outer, _, inner = _view(full_shape, axis)
        counts = [sz * outer * inner for sz in sizes]
        s = src[r]
        if self._use_p2p(kind, sum(counts), 2 if s.dtype == BF16 else 4):
            # hand-written NVLink kernel: exact chunks, placed in the final layout
            exact = not accumulate and dst[r].dtype == s.dtype
            target = dst[r] if exact else self._new(full_shape, s.dtype)
            push = self.cfg.p2p_push and exact
            fn = "hap_p2p_all_gather_push" if push else "hap_p2p_all_gather_v"
            self._p2p(fn, s, target, outer, inner, full_shape[axis], sizes,
                      16 if push else max(counts) * (2 if s.dtype == BF16 else 4))
            if not exact:
                self._copy(target, dst[r], self.caps[r], accumulate=accumulate)
            return
        direct = outer == 1 and not accumulate and dst[r].dtype == s.dtype
        target = dst[r] if direct else self._new((sum(counts),), s.dtype)
        carr = _lib.i64_array(counts)
        self._keep(carr)
        if kind == "grouped_broadcast":
            self._emit("hap_grouped_broadcast", self._comm(), s.ptr, target.ptr, carr, s.dtype,
                       self._sptr(), kernel=False)
        else:
            padded = self.cfg.gather == "padded"
            scratch = self._new((self.m * max(counts),), s.dtype) if padded else None
            self._emit("hap_all_gather_v", self._comm(), s.ptr, target.ptr, carr, s.dtype, int(padded),
                       scratch.ptr if scratch else None, self._sptr(), kernel=False)
        if not direct:
            # rank-ordered chunks [outer, size_k, inner] -> full [outer, E, inner]
            coff = offsets(counts)
            for k in range(self.m):
                if sizes[k] == 0:
                    continue
                chunk = Buf(target.tensor[coff[k]:coff[k + 1]] if target.tensor.numel() > 1 else target.tensor,
                            target.dtype, (outer, sizes[k], inner))
                self._block(chunk, (outer, sizes[k], inner), 0, dst[r], (outer, full_shape[axis], inner),
                            offs[k], sizes[k], self.caps[r], accumulate)

    def _coll_reduce_scatter(self, src: dict, dst: dict, axis: int, sizes: list, accumulate: int):
        """Partial full tensors -> summed shard ``rank`` along ``axis``."""
        g = self.group
        full_shape = src[g.local_ranks[0]].shape
        offs = offsets(sizes)
        outer, ext, inner = _view(full_shape, axis)
        if isinstance(g, LocalGroup):
            tmp = self._new(full_shape, F32)
            for k in range(self.m):
                self._copy(src[k], tmp, self.caps[k], accumulate=int(k > 0))
            for j in range(self.m):
                self._block(tmp, (outer, ext, inner), offs[j], dst[j], (outer, sizes[j], inner), 0,
                            sizes[j], self.caps[j], accumulate)
            return
        r = g.rank
        s = src[r]
        counts = [sz * outer * inner for sz in sizes]
        if self._use_p2p("reduce_scatter", sum(counts), 2 if s.dtype == BF16 else 4):
            exact = not accumulate and dst[r].dtype == s.dtype
            target = dst[r] if exact else self._new(dst[r].shape, s.dtype)
            if self.cfg.p2p_push:   # read the peers' partials in place (registered)
                self._p2p("hap_p2p_reduce_scatter_direct", s, target, outer, inner, ext, sizes, 16)
            else:
                self._p2p("hap_p2p_reduce_scatter_v", s, target, outer, inner, ext, sizes,
                          outer * ext * inner * (2 if s.dtype == BF16 else 4))
            if not exact:
                self._copy(target, dst[r], self.caps[r], accumulate=accumulate)
            return
        if outer == 1:
            send = s
        else:  # pack rank-ordered chunks
            send = self._new((sum(counts),), s.dtype)
            coff = offsets(counts)
            for k in range(self.m):
                if sizes[k]:
                    chunk = Buf(send.tensor[coff[k]:coff[k + 1]], s.dtype, (outer, sizes[k], inner))
                    self._block(s, (outer, ext, inner), offs[k], chunk, (outer, sizes[k], inner), 0,
                                sizes[k], self.caps[r])
        direct = not accumulate and dst[r].dtype == s.dtype
        target = dst[r] if direct else self._new(dst[r].shape, s.dtype)
        scratch = self._new((self.m * max(max(counts), 1),), s.dtype)
        carr = _lib.i64_array(counts)
        self._keep(carr)
        self._emit("hap_reduce_scatter_v", self._comm(), send.ptr, target.ptr, carr, s.dtype, scratch.ptr,
                   self._sptr(), kernel=False)
        if not direct:
            self._copy(target, dst[r], self.caps[r], accumulate=accumulate)

    def _coll_all_to_all(self, src: dict, src_shapes: list, dst: dict, d1: int, d2: int, sizes2: list,
                         accumulate: int):
        """Shards along d1 (all devices' shapes ``src_shapes``) -> shards along d2."""
        g = self.group
        sizes1 = [s[d1] for s in src_shapes]
        off1, off2 = offsets(sizes1), offsets(sizes2)
        if isinstance(g, LocalGroup):
            for j in range(self.m):
                for k in range(self.m):
                    # block of src_k (rows off1[k] of the full tensor along d1)
                    # restricted to device j's range along d2.
                    piece_shape = tuple(sizes2[j] if a == d2 else e for a, e in enumerate(src_shapes[k]))
                    piece = self._new(piece_shape, src[k].dtype)
                    self._block(src[k], _view(src_shapes[k], d2), off2[j], piece, _view(piece_shape, d2), 0,
                                sizes2[j], self.caps[j])
                    self._block(piece, _view(piece_shape, d1), 0, dst[j], _view(dst[j].shape, d1), off1[k],
                                sizes1[k], self.caps[j], accumulate)
            return
        r = g.rank
        s = src[r]
        send_shapes = [tuple(sizes2[k] if a == d2 else e for a, e in enumerate(s.shape)) for k in range(self.m)]
        send_counts = [int(math.prod(sh)) for sh in send_shapes]
        send = self._new((max(1, sum(send_counts)),), s.dtype)
        soff = offsets(send_counts)
        for k in range(self.m):
            if send_counts[k]:
                chunk = Buf(send.tensor[soff[k]:soff[k + 1]], s.dtype, send_shapes[k])
                self._block(s, _view(s.shape, d2), off2[k], chunk, _view(send_shapes[k], d2), 0, sizes2[k],
                            self.caps[r])
        recv_shapes = [tuple(sizes1[k] if a == d1 else e for a, e in enumerate(dst[r].shape)) for k in range(self.m)]
        recv_counts = [int(math.prod(sh)) for sh in recv_shapes]
        recv = self._new((max(1, sum(recv_counts)),), s.dtype)
        full = sum(int(math.prod(sh)) for sh in src_shapes)
        if self._use_p2p("all_to_all", full, 2 if s.dtype == BF16 else 4):
            # rank j's chunk for rank k lands at k's receive offset sum_{i<j} count(i -> k)
            def count(j, k):
                return int(math.prod(tuple(sizes2[k] if a == d2 else e for a, e in enumerate(src_shapes[j]))))
            dst_off = [sum(count(i, k) for i in range(r)) for k in range(self.m)]
            self._p2p_all_to_all(send, recv, soff[:-1], send_counts, dst_off)
        else:
            sarr, rarr = _lib.i64_array(send_counts), _lib.i64_array(recv_counts)
            self._keep(sarr)
            self._keep(rarr)
            self._emit("hap_all_to_all_v", self._comm(), send.ptr, sarr, recv.ptr, rarr, s.dtype, self._sptr(),
                       kernel=False)
        roff = offsets(recv_counts)
        for k in range(self.m):
            if recv_counts[k]:
                chunk = Buf(recv.tensor[roff[k]:roff[k + 1]], s.dtype, recv_shapes[k])
                self._block(chunk, _view(recv_shapes[k], d1), 0, dst[r], _view(dst[r].shape, d1), off1[k],
                            sizes1[k], self.caps[r], accumulate)

    def _use_p2p(self, kind: str, elements: int, esize: int, side: bool = False) -> bool:
        """Hand-written NVLink kernel (True) or NCCL (False) for one call site.

        A PeerGroup has only the kernels; ``gather`` forces one side.
        "auto" prices both with the reference cost model (cost_model.comm_time,
        cost_model.py:203) on the measured lines of each implementation
        (workloads.collective_fits: fit_linear over tools/coll_fit.py sweeps)
        and the plan's ratio row, and takes the cheaper; without measurements,
        the kernels for the gathers and reduce-scatters (exact uneven chunks in
        their final layout) and NCCL otherwise.  Without peer access between
        the GPUs, NCCL."""
        g = self.group
        if g.comm is None:
            return True
        if self.cfg.gather == "kernel":
            return True
        if self.cfg.gather in ("padded", "sendrecv", "nccl") or not self._peer_access():
            return False
        if side or getattr(self, "_emit_on", None) is not None:
            # side-stream call sites (SFB factor gathers, gradient buckets): the
            # fitted lines were measured with the compute stream idle and do not
            # predict these — measured at 2 GPUs, SFB with the push kernel 2,148
            # samples/s vs NCCL gathers 1,581; bucketed all-reduce over NCCL
            # 1,662 vs the two-shot kernel (32 CTAs) 1,003 — so gathers take the
            # kernel and all-reduces NCCL
            use = kind in ("all_gather", "grouped_broadcast")
            self.impl_choice.append((kind, elements * esize, "p2p" if use else "nccl", None, None))
            return use
        specs = self._impl_specs(esize)
        if specs is None:
            use = kind in ("all_gather", "grouped_broadcast", "reduce_scatter")
            self.impl_choice.append((kind, elements * esize, "p2p" if use else "nccl", None, None))
            return use
        from .cost_model import comm_time

        caps = [c or 148 for c in self.caps]   # no cap: the whole GPU
        row = tuple(self.cfg.ratios) if self.cfg.ratios else tuple(c / sum(caps) for c in caps)
        ins = Instruction("all_gather" if kind == "grouped_broadcast" else kind, "t", elements=int(elements))
        t_p2p, t_nccl = comm_time(ins, row, specs["p2p"]), comm_time(ins, row, specs["nccl"])
        use = t_p2p <= t_nccl
        self.impl_choice.append((kind, elements * esize, "p2p" if use else "nccl", t_p2p, t_nccl))
        return use

    def _impl_specs(self, esize: int):
        """ClusterSpecs carrying each implementation's fitted lines (or None)."""
        cache = self.__dict__.setdefault("_impl_spec_cache", {})
        if esize not in cache:
            from . import workloads
            from .cost_model import ClusterSpec

            caps = [c or 148 for c in self.caps]
            docs = {impl: workloads.impl_cluster_doc(caps, impl, esize) for impl in ("p2p", "nccl")}
            cache[esize] = None if any(d is None for d in docs.values()) else \
                {impl: ClusterSpec.from_dict(d) for impl, d in docs.items()}
        return cache[esize]

    def _peer_access(self) -> bool:
        """Every GPU this node's ranks use can map every other's memory (the
        peer-memory kernels need it); agreed across ranks once."""
        if "_peer_ok" not in self.__dict__:
            ok = True
            if not self.dry and torch.cuda.is_available():
                me = self.device.index if self.device.index is not None else torch.cuda.current_device()
                n = torch.cuda.device_count()
                ok = all(torch.cuda.can_device_access_peer(me, j) for j in range(n) if j != me)
            if self.group.distributed:
                ok = all(self.group.exchange(ok))
            self._peer_ok = ok
        return self._peer_ok

    def _p2p_tag(self) -> str:
        # one context (staging arena + flag epochs) per stream: calls on one
        # stream are ordered, calls on two streams must not share flags
        return "side" if self._emit_on is not None else "main"

    SIDE_P2P_CTAS = 32
    IN_PROCESS_P2P_CTAS = 16

    def _p2p_cap(self, tag: str) -> int:
        """Grid cap of a peer kernel: the rank's SM cap; on the side stream at
        most SIDE_P2P_CTAS, so a spinning side-stream kernel leaves the
        compute stream's persistent GEMM most of the GPU.  Ranks sharing one
        GPU (thread_peer_groups): at most IN_PROCESS_P2P_CTAS, because a
        rank's peer kernel spins while its partner may still be running a
        persistent SM-pair GEMM, whose CTAs (clusters of two on one TPC) must
        all become resident: the hardware may place the spinner's CTAs one
        per TPC, so with m ranks at most m x 16 TPCs are held, leaving the
        largest capped GEMM (ceil(148 / m / 2) TPCs) room on the 74."""
        cap = self.caps[self.group.rank] or 148
        if getattr(self.group, "in_process", False):
            return min(cap, self.IN_PROCESS_P2P_CTAS)
        return min(cap, self.SIDE_P2P_CTAS) if tag == "side" else cap

    def _register(self, tag: str, buf: Buf) -> dict:
        """A buffer every peer maps (push outputs, in-place partials): the
        device array of all ranks' pointers to it is filled in by
        _register_outputs once compilation is done."""
        reg: dict = {}
        self._p2p_regs.append((tag, buf, reg))
        return reg

    def _p2p(self, fn: str, send: Buf, recv: Buf, outer: int, inner: int, extent: int, sizes: list,
             arena_bytes: int):
        """Emit a peer-memory collective; the symmetric arena is created once
        compilation knows the largest staging need (same on every rank)."""
        r = self.group.rank
        dev = torch.tensor([list(sizes), offsets(sizes)[:-1]], dtype=torch.int64, device=self.device)
        self._keep(dev)
        tag = self._p2p_tag()
        self._p2p_bytes[tag] = max(self._p2p_bytes.get(tag, 0), arena_bytes)
        fn_ptr = getattr(self.lib, fn)
        stream = self._sptr()
        cap = self._p2p_cap(tag)
        sizes_ptr, offs_ptr = dev[0].data_ptr(), dev[1].data_ptr()
        if fn == "hap_p2p_all_gather_push":
            reg = self._register(tag, recv)
            total = outer * extent * inner
            args = lambda: (self._symm[tag], send.ptr, reg["dev"].data_ptr(), send.dtype, outer, inner,  # noqa: E731
                            extent, sizes_ptr, offs_ptr, total, cap, stream)
        elif fn == "hap_p2p_reduce_scatter_direct":
            reg = self._register(tag, send)
            mine = outer * sizes[r] * inner
            args = lambda: (self._symm[tag], reg["dev"].data_ptr(), recv.ptr, send.dtype, outer, inner,  # noqa: E731
                            extent, sizes_ptr, offs_ptr, mine, cap, stream)
        elif fn == "hap_p2p_all_gather_v":
            max_chunk = max(sizes) * outer * inner
            args = lambda: (self._symm[tag], send.ptr, recv.ptr, send.dtype, outer, inner, extent,  # noqa: E731
                            sizes_ptr, offs_ptr, max_chunk, cap, stream)
        else:
            args = lambda: (self._symm[tag], send.ptr, recv.ptr, send.dtype, outer, inner, extent,  # noqa: E731
                            sizes_ptr, offs_ptr, cap, stream)
        self._ops.append(Op(lambda: fn_ptr(*args()), (), fn, True,
                            meta=dict(send=send, recv=recv, outer=outer, inner=inner, extent=extent,
                                      sizes=list(sizes))))

    def _p2p_all_reduce(self, src: Buf, dst: Buf, n: int, stream_ptr=None):
        """Two-shot all-reduce kernel over registered buffers (src may be dst)."""
        tag = self._p2p_tag() if stream_ptr is None else "side"
        self._p2p_bytes[tag] = max(self._p2p_bytes.get(tag, 0), 16)
        reg_in = self._register(tag, src)
        reg_out = reg_in if dst is src else self._register(tag, dst)
        fn = self.lib.hap_p2p_all_reduce
        stream = stream_ptr if stream_ptr is not None else self._sptr()
        cap = self._p2p_cap(tag)
        dt = src.dtype
        self._ops.append(Op(lambda: fn(self._symm[tag], reg_in["dev"].data_ptr(), reg_out["dev"].data_ptr(), dt, n,
                                       cap, stream), (), "hap_p2p_all_reduce", True,
                            meta=dict(send=src, recv=dst, n=n)))

    def _p2p_all_to_all(self, send: Buf, recv: Buf, send_off: list, counts: list, dst_off: list):
        tag = self._p2p_tag()
        self._p2p_bytes[tag] = max(self._p2p_bytes.get(tag, 0), 16)
        reg = self._register(tag, recv)
        dev = torch.tensor([list(send_off), list(counts), list(dst_off)], dtype=torch.int64, device=self.device)
        self._keep(dev)
        fn = self.lib.hap_p2p_all_to_all
        stream = self._sptr()
        cap = self._p2p_cap(tag)
        most = max(max(counts), 1)
        self._ops.append(Op(lambda: fn(self._symm[tag], send.ptr, reg["dev"].data_ptr(), send.dtype,
                                       dev[0].data_ptr(), dev[1].data_ptr(), dev[2].data_ptr(), most, cap, stream),
                            (), "hap_p2p_all_to_all", True,
                            meta=dict(send=send, recv=recv, send_off=list(send_off), counts=list(counts),
                                      dst_off=list(dst_off))))

    def _create_symm(self):
        if not self._p2p_bytes or self.dry:
            return
        g = self.group
        for tag in sorted(self._p2p_bytes):   # same order on every rank
            ctx = ctypes.c_void_p()
            check(self.lib.hap_symm_create(ctypes.byref(ctx), int(self._p2p_bytes[tag]), g.rank, g.m),
                  "hap_symm_create")
            self._symm[tag] = ctx
            if getattr(g, "in_process", False):
                bases = g.exchange(int(self.lib.hap_symm_local_base(ctx) or 0))
                check(self.lib.hap_symm_open_local(ctx, _lib.i64_array(bases)), "hap_symm_open_local")
            else:
                handle = ctypes.create_string_buffer(64)
                check(self.lib.hap_symm_handle(ctx, handle), "hap_symm_handle")
                handles = g.exchange(bytes(handle.raw))
                check(self.lib.hap_symm_open(ctx, b"".join(handles)), "hap_symm_open")
        self._register_outputs()

    def _register_outputs(self):
        """Map every registered buffer (push outputs, in-place partials,
        all-reduce operands) into every peer: one exchange for all of them —
        (IPC handle, allocation base, offset) triples across processes, plain
        device pointers inside one process."""
        if not self._p2p_regs:
            return
        g = self.group
        if getattr(g, "in_process", False):
            everyone = g.exchange([buf.ptr for _, buf, _ in self._p2p_regs])
            for i, (_, _, reg) in enumerate(self._p2p_regs):
                reg["dev"] = torch.tensor([everyone[p][i] for p in range(g.m)], dtype=torch.int64, device=self.device)
                self._keep(reg["dev"])
            return
        mine = []
        for tag, buf, _ in self._p2p_regs:
            h = ctypes.create_string_buffer(64)
            base, off = ctypes.c_int64(), ctypes.c_int64()
            check(self.lib.hap_p2p_buffer_handle(self._symm[tag], buf.ptr, h, ctypes.byref(base), ctypes.byref(off)),
                  "hap_p2p_buffer_handle")
            mine.append((bytes(h.raw), base.value, off.value))
        everyone = g.exchange(mine)
        if len({len(x) for x in everyone}) != 1:
            raise ExecutionError(f"ranks registered {[len(x) for x in everyone]} peer-memory buffers: their "
                                 "collective implementation choices disagree")
        for i, (tag, buf, reg) in enumerate(self._p2p_regs):
            handles = b"".join(everyone[p][i][0] for p in range(g.m))
            bases = _lib.i64_array([everyone[p][i][1] for p in range(g.m)])
            offs = _lib.i64_array([everyone[p][i][2] for p in range(g.m)])
            ptrs = (ctypes.c_void_p * g.m)()
            check(self.lib.hap_p2p_buffer_open(self._symm[tag], buf.ptr, handles, bases, offs, ptrs),
                  "hap_p2p_buffer_open")
            reg["dev"] = torch.tensor([int(p or 0) for p in ptrs], dtype=torch.int64, device=self.device)
            self._keep(reg["dev"])

    def _batch_gemms(self, ops: list) -> list:
        """Merge runs of consecutive matmul launches into hap_matmul_batch
        launches: matmuls adding into one output (the adjoint contributions of
        an activation with several consumers) become one K-concatenated GEMM;
        independent matmuls sharing an input (Q/K/V projections, their weight
        gradients) share one persistent launch.  An op joins a group only if
        nothing it reads or writes is touched by the ops it is moved past."""
        out: list = []
        i = 0
        while i < len(ops):
            if ops[i].gemm is None:
                out.append(ops[i])
                i += 1
                continue
            j = i
            while j < len(ops) and ops[j].gemm is not None:
                j += 1
            out.extend(self._group_run(ops[i:j]))
            i = j
        return out

    def _group_run(self, run: list) -> list:
        def reads(g):
            r = {g["A"], g["B"]} | ({g["R"], g["R2"]} - {None})
            if g["accumulate"]:
                r.add(g["C"])
            return r

        def writes(g):
            return {g["C"], g["Y"], g["Z"]} - {None}

        def compatible(a, b):
            keys = ("transA", "transB", "in_dt", "out_dt", "cap", "stream")
            return all(a[k] == b[k] for k in keys)

        placed = [False] * len(run)
        result = []
        for i, op in enumerate(run):
            if placed[i]:
                continue
            g0 = op.gemm
            members = [i]
            placed[i] = True
            sum_k = False
            for j in range(i + 1, len(run)):
                if placed[j]:
                    continue
                gj = run[j].gemm
                if not compatible(g0, gj):
                    continue
                same_out = gj["C"] == g0["C"]
                if same_out:
                    # a K-concatenated sum: later terms plain accumulates; the
                    # first term's epilogue (at most an addend) applies to the sum
                    if not (gj["accumulate"] and (gj["M"], gj["N"], gj["ldc"]) == (g0["M"], g0["N"], g0["ldc"])):
                        continue
                    if gj["epi"] != _lib.EPI_NONE or g0["epi"] not in (_lib.EPI_NONE, _lib.EPI_ADD):
                        continue
                    if len(members) > 1 and not sum_k:
                        continue
                elif sum_k or any(writes(run[m].gemm) & (reads(gj) | writes(gj)) for m in members) or \
                        any(writes(gj) & reads(run[m].gemm) for m in members):
                    continue
                # the ops skipped over (not in the group, not yet placed) must not conflict
                between = [k for k in range(i + 1, j) if not placed[k] and k not in members]
                conflict = False
                for k in between:
                    gk = run[k].gemm
                    if writes(gk) & reads(gj) or writes(gj) & reads(gk) or writes(gk) & writes(gj):
                        conflict = True
                        break
                if conflict:
                    continue
                if same_out:
                    sum_k = True
                members.append(j)
                placed[j] = True
                if len(members) == 4:
                    break
            if len(members) == 1:
                result.append(op)
                continue
            descs = (_lib.GemmDesc * len(members))()
            for slot, m in enumerate(members):
                self._fill_desc(descs[slot], run[m].gemm)
            self._keep(descs)
            result.append(Op(self.lib.hap_matmul_batch, (descs, len(members), int(sum_k), g0["in_dt"],
                                                         g0["out_dt"], g0["cap"], g0["stream"]),
                             "hap_matmul_batch", True,
                             dict(g0, members=[run[m].gemm for m in members], sum_k=sum_k)))
        return result

    # Non-GEMM launches whose every buffer is a direct pointer argument (the
    # hazard scan of _offload_wgrad can see what they touch).
    _DIRECT_OPS = frozenset({"hap_unary", "hap_unary_grad", "hap_binary", "hap_mul_grad", "hap_swish_fwd",
                             "hap_swish_bwd", "hap_gate_fwd", "hap_gate_bwd", "hap_axpy", "hap_copy_block",
                             "hap_unreduce", "hap_fill", "hap_reduce"})

    @staticmethod
    def _gemm_ranges(g: dict) -> tuple[list, list]:
        """(read, write) byte ranges of a GEMM record's members."""
        rd, wr = [], []
        for m in g.get("members", [g]):
            ein = 2 if m["in_dt"] == BF16 else 4
            eout = 2 if m["out_dt"] == BF16 else 4
            rd.append((m["A"], (m["K"] if m["transA"] else m["M"]) * m["lda"] * ein))
            rd.append((m["B"], (m["N"] if m["transB"] else m["K"]) * m["ldb"] * ein))
            for p, ld in (("R", "ldr"), ("R2", "ldr2")):
                if m[p]:
                    rd.append((m[p], m["M"] * m[ld] * 2))
            c = (m["C"], m["M"] * m["ldc"] * eout)
            wr.append(c)
            if m["accumulate"]:
                rd.append(c)
            for p, ld in (("Y", "ldy"), ("Z", "ldz")):
                if m[p]:
                    wr.append((m[p], m["M"] * m[ld] * 2))
        return [(a, a + n) for a, n in rd], [(a, a + n) for a, n in wr]

    def _offload_wgrad(self, ops: list) -> list:
        """Move the parameter-gradient GEMMs (dW = X^T.dY into a source's fp32
        gradient) onto a side stream.  They depend only on finished forward
        activations and finished output gradients, and nothing on the
        activation-gradient chain reads their results, so their tiles fill the
        SMs the chain's launches leave idle (each launch's partial last wave,
        prologue and epilogue tail).  Fork: an event on the compute stream
        right before the GEMM.  Join (compute stream waits for the side
        stream) before the first later op that might touch a moved GEMM's
        buffers — GEMMs by their descriptors, direct-pointer kernels by their
        pointer arguments, and conservatively before every other op (events,
        collectives, the SGD table launch) — and at the end."""
        grad_ranges = []
        for (did, r), b in self.grads.items():
            if did in self.source_dids:
                grad_ranges.append((b.ptr, b.ptr + max(1, b.numel) * (4 if b.dtype == F32 else 2)))

        def inside(p, ranges):
            return isinstance(p, int) and any(lo <= p < hi for lo, hi in ranges)

        def overlaps(a, b):
            return any(lo < hi2 and lo2 < hi for lo, hi in a for lo2, hi2 in b)

        def candidate(op):
            g = op.gemm
            if g is None or not op.kernel:
                return False
            ms = g.get("members", [g])
            return all(m["epi"] == _lib.EPI_NONE and m["out_dt"] == F32 and inside(m["C"], grad_ranges)
                       and not m["Y"] and not m["Z"] for m in ms)

        side = None
        out: list = []
        active_rd, active_wr = [], []      # ranges of the moved GEMMs since the last join
        prev_moved = False
        moved = forks = joins = 0

        def join():
            nonlocal joins
            ev = self._event()
            self._keep(ev)
            out.append(Op(ev.record, (side,), "event.record", False))
            out.append(Op(self.stream.wait_event, (ev,), "stream.wait_event", False))
            joins += 1

        for op in ops:
            if candidate(op):
                if side is None:
                    side = self._stream()
                    self.wgrad_stream = side
                if not prev_moved:
                    ev = self._event()
                    self._keep(ev)
                    out.append(Op(ev.record, (self.stream,), "event.record", False))
                    out.append(Op(side.wait_event, (ev,), "stream.wait_event", False))
                    forks += 1
                g = op.gemm
                sp = side.cuda_stream
                op.args = op.args[:-1] + (sp,)
                g["stream"] = sp
                for m in g.get("members", []):
                    m["stream"] = sp
                rd, wr = self._gemm_ranges(g)
                active_rd += rd
                active_wr += wr
                out.append(op)
                prev_moved = True
                moved += 1
                continue
            prev_moved = False
            if active_wr:
                if op.gemm is not None:
                    rd, wr = self._gemm_ranges(op.gemm)
                    hazard = overlaps(wr, active_rd + active_wr) or overlaps(rd, active_wr)
                elif op.what in self._DIRECT_OPS:
                    hazard = any(inside(a, active_rd + active_wr) for a in op.args)
                else:
                    hazard = True
                if hazard:
                    join()
                    active_rd, active_wr = [], []
            out.append(op)
        if active_wr:
            join()
        self.wgrad_stats = (moved, forks, joins)
        return out

    def _keep(self, obj):
        self.__dict__.setdefault("_keepalive", []).append(obj)

    # ------------------------------------------------------------------ forward
    def _compile_forward(self):
        self._ops = self.ops_fwd
        self._find_chains()
        # activations that sufficient-factor broadcasting will gather: with a
        # side stream, gather each as soon as it is produced
        early = set()
        if self._sfb_overlap() and os.environ.get("HAP_DBG_SFB_FWD", "1") == "1":
            early = {u.operands[0] for uses in self.sfb.values() for u in uses}
            for d in sorted(early & self.source_dids):
                self._sfb_factor(d, {r: self.bufs[(d, r)] for r in self.group.local_ranks})
        skip: set = set()
        for idx, ins in enumerate(self.program.instrs):
            if idx in skip:
                continue
            chain = self.chains.get(idx)
            if chain is not None:
                self._forward_chain(chain)
                skip.update(chain["members"][1:])
                outs = [self.program.instrs[i].output for i in chain["members"]]
            else:
                self._forward_instr(ins)
                outs = [ins.output]
            for d in outs:
                if d in early and d not in self.source_dids:
                    self._sfb_factor(d, {r: self.bufs[(d, r)] for r in self.group.local_ranks})
        self._loss_closure()

    def _find_chains(self):
        """Elementwise chains fused into one kernel (forward and backward):
        swish  y = f(x), z = x*y   and   gate  p = a*b, q = f(p), o = q*c,
        consecutive compute instructions over one dtype and shape.  The
        backward fusion additionally needs each chain-internal tensor (y; p
        and q) to have no consumer outside the chain."""
        self.chains: dict = {}
        self.chain_of: dict = {}
        if not self.cfg.fuse_elementwise:
            return
        consumers: dict = {}
        for ins in self.program.instrs:
            for d in ins.operands:
                consumers.setdefault(d, []).append(ins)
        compute = [(i, ins) for i, ins in enumerate(self.program.instrs) if ins.kind not in SOURCE_KINDS]
        L = self.group.local_ranks

        def uniform(dids):
            dts = {self.dtypes[d] for d in dids}
            shapes = {tuple(self.shapes[d][r]) for d in dids for r in L}
            return len(dts) == 1 and len(shapes) == 1

        used: set = set()
        for pos, (i, u) in enumerate(compute):
            if i in used:
                continue
            nxt = compute[pos + 1] if pos + 1 < len(compute) else None
            nxt2 = compute[pos + 2] if pos + 2 < len(compute) else None
            # swish at a unary instruction
            if u.kind == "elemwise_unary" and nxt is not None:
                j, bm = nxt
                x, y = u.operands[0], u.output
                if (bm.kind == "elemwise_binary" and bm.tag == "mul" and set(bm.operands) == {x, y} and x != y
                        and uniform([x, y, bm.output])):
                    c = {"kind": "swish", "members": [i, j], "u": u, "b": bm, "x": x, "y": y, "z": bm.output,
                         "bwd": [ins.output for ins in consumers.get(y, [])] == [bm.output]}
                    self.chains[i] = c
                    self.chain_of[j] = c
                    self.chain_of[i] = c
                    used.update((i, j))
                    continue
            # gate at a mul instruction
            if (u.kind == "elemwise_binary" and u.tag == "mul" and nxt is not None and nxt2 is not None):
                (j, un), (k, b2) = nxt, nxt2
                a_, b_ = u.operands
                p_ = u.output
                if (un.kind == "elemwise_unary" and un.operands[0] == p_ and b2.kind == "elemwise_binary"
                        and b2.tag == "mul" and un.output in b2.operands):
                    q_ = un.output
                    c_ = b2.operands[1] if b2.operands[0] == q_ else b2.operands[0]
                    dids = [a_, b_, c_, p_, q_, b2.output]
                    if len({a_, b_, c_, p_, q_}) == 5 and uniform(dids):
                        c = {"kind": "gate", "members": [i, j, k], "b1": u, "u": un, "b2": b2, "a": a_, "b": b_,
                             "c": c_, "p": p_, "q": q_, "o": b2.output,
                             "bwd": ([ins.output for ins in consumers.get(p_, [])] == [q_]
                                     and [ins.output for ins in consumers.get(q_, [])] == [b2.output])}
                        self.chains[i] = c
                        for m in (i, j, k):
                            self.chain_of[m] = c
                        used.update((i, j, k))

    def _forward_chain(self, c: dict):
        L = self.group.local_ranks
        B = lambda d, r: self.bufs[(d, r)]  # noqa: E731
        for r in L:
            if c["kind"] == "swish":
                x, y, z = B(c["x"], r), B(c["y"], r), B(c["z"], r)
                op = self._producer_gemm(x.ptr) if self.cfg.fuse_swish_fwd else None
                if op is not None and op.gemm["accumulate"] == 0 and self._gemm_fusable(op.gemm) \
                        and self._fusable_buf(x, y, z):
                    op.gemm.update(epi=_lib.EPI_SWISH, epi_tag=_lib.UNARY_TAGS[c["u"].tag], Y=y.ptr,
                                   ldy=y.shape[1], Z=z.ptr, ldz=z.shape[1])
                    self._sync_desc(op)
                    continue
                self._emit("hap_swish_fwd", _lib.UNARY_TAGS[c["u"].tag], x.ptr, y.ptr, z.ptr, x.dtype, x.numel,
                           self.caps[r], self._sptr())
            else:
                a, b, cc = B(c["a"], r), B(c["b"], r), B(c["c"], r)
                p, q, o = B(c["p"], r), B(c["q"], r), B(c["o"], r)
                self._emit("hap_gate_fwd", _lib.UNARY_TAGS[c["u"].tag], a.ptr, b.ptr, cc.ptr, p.ptr, q.ptr, o.ptr,
                           a.dtype, a.numel, self.caps[r], self._sptr())

    def _forward_instr(self, ins: Instruction):
        k = ins.kind
        if k in SOURCE_KINDS:
            return  # bound by load()/feed()
        L = self.group.local_ranks
        out = {r: self.bufs[(ins.output, r)] for r in L}
        src = [{r: self.bufs[(d, r)] for r in L} for d in ins.operands]
        if k == "matmul":
            for r in L:
                self._gemm(src[0][r], False, src[1][r], False, out[r], self.caps[r], 0)
        elif k == "elemwise_unary":
            for r in L:
                self._emit("hap_unary", _lib.UNARY_TAGS[ins.tag], src[0][r].ptr, src[0][r].dtype,
                           out[r].ptr, out[r].dtype, out[r].numel, self.caps[r], self._sptr())
        elif k == "elemwise_binary":
            for r in L:
                a, b = src[0][r], src[1][r]
                if ins.tag == "add" and ins.operands[0] != ins.operands[1] and self._fusable_buf(a, b, out[r]):
                    # out = C + R folded into the epilogue of the GEMM that produced C
                    op, other = self._producer_gemm(b.ptr), a
                    if op is None:
                        op, other = self._producer_gemm(a.ptr), b
                    if op is not None and op.gemm["accumulate"] == 0 and self._gemm_fusable(op.gemm):
                        op.gemm.update(epi=_lib.EPI_ADD2, R=other.ptr, ldr=other.shape[1], Y=out[r].ptr,
                                       ldy=out[r].shape[1])
                        self._sync_desc(op)
                        continue
                in_dt = BF16 if a.dtype == BF16 and b.dtype == BF16 else F32
                a, b = self._as(a, in_dt, self.caps[r]), self._as(b, in_dt, self.caps[r])
                self._emit("hap_binary", _lib.BINARY_TAGS[ins.tag], a.ptr, b.ptr, in_dt, out[r].ptr,
                           out[r].dtype, out[r].numel, self.caps[r], self._sptr())
        elif k == "identity":
            for r in L:
                self._copy(src[0][r], out[r], self.caps[r])
        elif k == "reduce":
            for r in L:
                x = src[0][r]
                self._reduce(x, ins.dims, out[r], self.caps[r], 0)
        elif k == "all_reduce":
            self._coll_all_reduce(src[0], out, 0)
        elif k in ("all_gather", "grouped_broadcast"):
            self._coll_all_gather(src[0], self.shapes[ins.operands[0]], out, ins.axis, 0, k)
        elif k == "reduce_scatter":
            self._coll_reduce_scatter(src[0], out, ins.axis, self._sizes(ins.ref, ins.axis), 0)
        elif k == "all_to_all":
            self._coll_all_to_all(src[0], self.shapes[ins.operands[0]], out, ins.axis, ins.axis2,
                                  self._sizes(ins.ref, ins.axis2), 0)
        else:
            raise ExecutionError(f"unsupported instruction kind {k!r}")

    def _reduce(self, x: Buf, dims, y: Buf, cap: int, accumulate: int):
        mask = 0
        for d in dims:
            mask |= 1 << d
        shape = _lib.i64_array(x.shape) if x.shape else _lib.i64_array([1])
        self._keep(shape)
        if y.dtype != F32:
            raise ExecutionError("reduce outputs are fp32")
        self._emit("hap_reduce", x.ptr, x.dtype, shape, len(x.shape), mask, y.ptr, y.dtype, accumulate,
                   cap, self._sptr())

    def _loss_closure(self):
        """interpreter.py:193 — full form if realised, else all-reduce the partial."""
        L = self.group.local_ranks
        loss = self.program.loss
        if f"{loss}@full" in self.shapes:
            for r in L:
                self._copy(self.bufs[(f"{loss}@full", r)], self.loss_buf[r], self.caps[r])
        elif f"{loss}@partial" in self.shapes:
            self._coll_all_reduce({r: self.bufs[(f"{loss}@partial", r)] for r in L}, self.loss_buf, 0)
        else:
            raise ExecutionError(f"program realizes no property of the loss tensor {loss!r}")

    # ------------------------------------------------------------------ backward
    def _grad(self, did: str, r: int) -> Buf:
        key = (did, r)
        if key not in self.grads:
            fwd = self.bufs[key]
            dt = F32 if (fwd.dtype == F32 or did in self.source_dids) else fwd.dtype
            self.grads[key] = self._new(fwd.shape, dt)
        return self.grads[key]

    def _compile_backward(self):
        self._ops = self.ops_bwd
        L = self.group.local_ranks
        loss = self.program.loss
        written: set[str] = set()   # grads that already hold a contribution
        self._written = written

        self._pending: dict = {}    # (did, r) -> Buf: deferred first contribution (a plain copy)

        def contrib(did: str, fuse_ok: bool = False) -> int:
            """accumulate flag for the next contribution to grad(did).  A
            deferred copy into grad(did) is emitted first unless the caller
            folds it into its own launch (fuse_ok: a GEMM epilogue addend)."""
            if not fuse_ok:
                self._flush_pending(did)
            acc = int(did in written)
            written.add(did)
            return acc

        if f"{loss}@full" in self.shapes:
            seed_did, seed_val = f"{loss}@full", 1.0 / self.m
        else:
            seed_did, seed_val = f"{loss}@partial", 1.0
        if not self.req.get(seed_did, False):
            self._finish_update(written)
            return
        for r in L:
            gb = self._grad(seed_did, r)
            self._emit("hap_fill", gb.ptr, gb.dtype, seed_val, max(1, gb.numel), self._sptr())
        written.add(seed_did)

        self._grad_ready_at: dict = {}
        self.overlapped: set = set()
        self._count_contributions(seed_did)
        self._flat_grads()
        index = {id(ins): i for i, ins in enumerate(self.program.instrs)}
        handled: set = set()
        for ins in reversed(self.program.instrs):
            if ins.output not in written or ins.kind in SOURCE_KINDS:
                continue
            need = [self.req[d] for d in ins.operands]
            if not any(need):
                continue
            idx = index[id(ins)]
            if idx in handled:
                continue
            chain = self.chain_of.get(idx)
            if chain is not None and chain["bwd"] and idx == chain["members"][-1] and self._chain_bwd_ok(chain):
                self._adjoint_chain(chain, contrib)
                handled.update(chain["members"])
                for d in self._chain_inputs(chain):
                    if d in self.source_dids:
                        self._grad_ready_at[d] = len(self._ops)
                continue
            self._adjoint(ins, need, contrib)
            for d in ins.operands:
                if d in self.source_dids:
                    self._grad_ready_at[d] = len(self._ops)
        self._flush_pending()
        self._emit_sfb_pending()
        self._overlap_grad_sync()
        self._finish_update(written)

    def _flush_pending(self, did: str | None = None):
        """Emit deferred gradient copies (of ``did``, or all)."""
        for key in [k for k in self._pending if did is None or k[0] == did]:
            src = self._pending.pop(key)
            self._copy(src, self._grad(key[0], key[1]), self.caps[key[1]])

    def _defer_copy(self, did: str, dy: dict) -> bool:
        """First contribution to grad(did) is a plain copy of dy (an add's
        adjoint) and more contributions follow: defer it, so a GEMM that adds
        into grad(did) next reads dy as its epilogue addend instead."""
        L = self.group.local_ranks
        if not self.cfg.fuse_epilogue or did in self._written or self._n_contrib.get(did, 0) < 2 \
                or did in self.source_dids:
            return False
        if any(not self._fusable_buf(dy[r], self.bufs[(did, r)]) or self.dtypes[did] != BF16 for r in L):
            return False
        for r in L:
            self._grad(did, r)
            self._pending[(did, r)] = dy[r]
        self._written.add(did)
        return True

    def _chain_bwd_ok(self, c: dict) -> bool:
        """The fused adjoint keeps one dtype: every input gradient must be
        stored in the chain's working precision (sources keep fp32 grads)."""
        dt = self.dtypes[self._chain_inputs(c)[0]]
        for d in self._chain_inputs(c):
            if self.req[d] and (d in self.source_dids and dt != F32):
                return False
        return all(self.dtypes[d] == dt for d in self._chain_inputs(c))

    @staticmethod
    def _chain_inputs(c: dict) -> list:
        return [c["x"]] if c["kind"] == "swish" else [c["a"], c["b"], c["c"]]

    def _adjoint_chain(self, c: dict, contrib):
        """Fused adjoint of a whole chain: contributions to the chain inputs
        only (the internal gradients dy / dq, dp are never materialised)."""
        L = self.group.local_ranks
        tag = _lib.UNARY_TAGS[c["u"].tag]
        self._flush_pending(c["z"] if c["kind"] == "swish" else c["o"])
        if c["kind"] == "swish":
            if not self.req[c["x"]]:
                return
            acc = contrib(c["x"])
            for r in L:
                x, y = self.bufs[(c["x"], r)], self.bufs[(c["y"], r)]
                dz, dx = self.grads[(c["z"], r)], self._grad(c["x"], r)
                # dx (+)= swish'(dz) folded into the epilogue of the GEMM that produced dz
                op = self._producer_gemm(dz.ptr)
                if op is not None and op.gemm["accumulate"] == 0 and acc == 0 and self._n_contrib.get(c["z"]) == 1 \
                        and c["z"] not in self.aliased and self._gemm_fusable(op.gemm) \
                        and self._fusable_buf(x, y, dz, dx):
                    op.gemm.update(epi=_lib.EPI_SWISH_BWD, epi_tag=tag, C=dx.ptr, ldc=dx.shape[1], R=x.ptr,
                                   ldr=x.shape[1], R2=y.ptr, ldr2=y.shape[1])
                    self._sync_desc(op)
                    continue
                self._emit("hap_swish_bwd", tag, x.ptr, y.ptr, dz.ptr, dx.ptr, x.dtype, x.numel, acc, self.caps[r],
                           self._sptr())
            return
        flags = {}
        for key in ("a", "b", "c"):
            flags[key] = contrib(c[key]) if self.req[c[key]] else 0
        for r in L:
            bf = lambda d: self.bufs[(d, r)]  # noqa: E731
            grad = lambda key: self._grad(c[key], r).ptr if self.req[c[key]] else None  # noqa: E731
            a = bf(c["a"])
            self._emit("hap_gate_bwd", tag, a.ptr, bf(c["b"]).ptr, bf(c["c"]).ptr, bf(c["p"]).ptr, bf(c["q"]).ptr,
                       self.grads[(c["o"], r)].ptr, grad("a"), grad("b"), grad("c"), a.dtype, a.numel, flags["a"],
                       flags["b"], flags["c"], self.caps[r], self._sptr())

    def _count_contributions(self, seed_did: str):
        """How many adjoint contributions each gradient will receive (a dry
        run of the reverse pass), so a gradient that receives exactly one
        plain copy can alias its source instead of being copied."""
        live = {seed_did}
        self._n_contrib: dict = {}
        for ins in reversed(self.program.instrs):
            if ins.output not in live or ins.kind in SOURCE_KINDS:
                continue
            need = [self.req[d] for d in ins.operands]
            if not any(need):
                continue
            operands = ins.operands
            if ins.kind == "elemwise_binary" and ins.tag == "mul" and operands[0] == operands[1]:
                operands = operands[:1]
            for d, nd in zip(operands, need):
                if nd:
                    self._n_contrib[d] = self._n_contrib.get(d, 0) + 1
                    live.add(d)

    def _alias_grad(self, did: str, dy: dict) -> bool:
        """Give grad(did) the buffers of dy when dy is its only contribution
        (dy is complete and never written again once its adjoint runs)."""
        L = self.group.local_ranks
        # sources are excluded: their gradients are synchronised in place
        if did in self.source_dids or self._n_contrib.get(did) != 1 or any((did, r) in self.grads for r in L):
            return False
        if any(dy[r].dtype != (F32 if (self.dtypes[did] == F32 or did in self.source_dids) else self.dtypes[did])
               for r in L):
            return False
        for r in L:
            self.grads[(did, r)] = dy[r]
        self._written.add(did)
        self.aliased.add(did)
        return True

    def _adjoint(self, ins: Instruction, need: list, contrib):
        L = self.group.local_ranks
        k = ins.kind
        self._flush_pending(ins.output)
        dy = {r: self.grads[(ins.output, r)] for r in L}
        x = [{r: self.bufs[(d, r)] for r in L} for d in ins.operands]
        ops = ins.operands
        if k == "matmul":
            if need[0]:
                acc = contrib(ops[0], fuse_ok=True)
                for r in L:     # dA = dC . B^T (+ a deferred copy as the epilogue addend)
                    pend = self._pending.get((ops[0], r))
                    g = self._grad(ops[0], r)
                    if pend is not None:
                        self._gemm(dy[r], False, x[1][r], True, g, self.caps[r], 0, addend=pend)
                        if self._gemm_fusable(dict(self._ops[-1].gemm, epi=_lib.EPI_NONE)):
                            del self._pending[(ops[0], r)]
                            continue
                        self._ops.pop()      # not fusable here: copy first, then accumulate
                        self._flush_pending(ops[0])
                    self._gemm(dy[r], False, x[1][r], True, g, self.caps[r], acc)
            if need[1]:
                if ops[1] in self.sfb:
                    self._sfb_weight_grad(ins, contrib)
                else:
                    acc = contrib(ops[1])
                    for r in L:     # dB = A^T . dC
                        self._gemm(x[0][r], True, dy[r], False, self._grad(ops[1], r), self.caps[r], acc)
        elif k == "elemwise_unary":
            acc = contrib(ops[0])
            tag = _lib.UNARY_TAGS[ins.tag]
            for r in L:
                xb, yb = x[0][r], self.bufs[(ins.output, r)]
                if xb.dtype != yb.dtype:
                    xb = self._as(xb, yb.dtype, self.caps[r])
                g = self._grad(ops[0], r)
                self._emit("hap_unary_grad", tag, xb.ptr, yb.ptr, yb.dtype, dy[r].ptr, dy[r].dtype,
                           g.ptr, g.dtype, g.numel, acc, self.caps[r], self._sptr())
        elif k == "identity":
            if self._alias_grad(ops[0], dy):
                return
            acc = contrib(ops[0])
            for r in L:
                self._copy(dy[r], self._grad(ops[0], r), self.caps[r], accumulate=acc)
        elif k == "elemwise_binary":
            if ins.tag == "add":
                for i in (0, 1):
                    if need[i] and not (ops[0] != ops[1] and self._alias_grad(ops[i], dy)):
                        if ops[0] != ops[1] and self._defer_copy(ops[i], dy):
                            continue
                        acc = contrib(ops[i])
                        for r in L:
                            self._copy(dy[r], self._grad(ops[i], r), self.caps[r], accumulate=acc)
            else:
                same = ops[0] == ops[1]
                if same:
                    acc = contrib(ops[0])
                    for r in L:
                        a = x[0][r]
                        g = self._grad(ops[0], r)
                        self._emit("hap_mul_grad", a.ptr, a.ptr, a.dtype, dy[r].ptr, dy[r].dtype, g.ptr,
                                   g.ptr, g.dtype, g.numel, acc, self.caps[r], self._sptr())
                elif need[0] and need[1] and (ops[0] in self._written) == (ops[1] in self._written):
                    # both adjoints in one pass over dy, a and b
                    acc = contrib(ops[0])
                    contrib(ops[1])
                    for r in L:
                        a, b = x[0][r], x[1][r]
                        ga, gb = self._grad(ops[0], r), self._grad(ops[1], r)
                        if a.dtype != b.dtype or ga.dtype != gb.dtype:
                            raise ExecutionError("mixed-precision mul operands")
                        self._emit("hap_mul_grad", a.ptr, b.ptr, a.dtype, dy[r].ptr, dy[r].dtype, ga.ptr,
                                   gb.ptr, ga.dtype, ga.numel, acc, self.caps[r], self._sptr())
                else:
                    for i in (0, 1):
                        if not need[i]:
                            continue
                        acc = contrib(ops[i])
                        for r in L:
                            other = x[1 - i][r]
                            g = self._grad(ops[i], r)
                            # d(a*b)/da = b : mul_grad with only the `da` output
                            self._emit("hap_mul_grad", other.ptr, other.ptr, other.dtype, dy[r].ptr,
                                       dy[r].dtype, g.ptr, None, g.dtype, g.numel, acc, self.caps[r],
                                       self._sptr())
        elif k == "reduce":
            acc = contrib(ops[0])
            mask = 0
            for d in ins.dims:
                mask |= 1 << d
            for r in L:
                xs = x[0][r].shape
                shape = _lib.i64_array(xs) if xs else _lib.i64_array([1])
                self._keep(shape)
                g = self._grad(ops[0], r)
                self._emit("hap_unreduce", dy[r].ptr, dy[r].dtype, shape, len(xs), mask, g.ptr, g.dtype,
                           acc, self.caps[r], self._sptr())
        elif k == "all_reduce":          # AR -> Id : adjoint is all-reduce
            acc = contrib(ops[0])
            self._coll_all_reduce(dy, {r: self._grad(ops[0], r) for r in L}, acc)
        elif k in ("all_gather", "grouped_broadcast"):   # AG(d) -> Id : reduce-scatter
            acc = contrib(ops[0])
            self._coll_reduce_scatter(dy, {r: self._grad(ops[0], r) for r in L}, ins.axis,
                                      self._sizes(ins.ref, ins.axis), acc)
        elif k == "reduce_scatter":      # AR -> AG(d) : all-gather
            acc = contrib(ops[0])
            for r in L:
                self._grad(ops[0], r)
            self._coll_all_gather(dy, self.shapes[ins.output], {r: self.grads[(ops[0], r)] for r in L},
                                  ins.axis, acc, "all_gather")
        elif k == "all_to_all":          # AG(d1) -> AG(d2) : all-to-all back
            acc = contrib(ops[0])
            for r in L:
                self._grad(ops[0], r)
            self._coll_all_to_all(dy, self.shapes[ins.output], {r: self.grads[(ops[0], r)] for r in L},
                                  ins.axis2, ins.axis, self._sizes(ins.ref, ins.axis), acc)
        else:
            raise ExecutionError(f"unsupported instruction kind {k!r}")

    # ------------------------------------------------------------------ gradient sync
    def _plan_sfb(self):
        """Pick sufficient-factor broadcasting for replicated parameters whose
        every use is a row-sharded matmul (x@shard0 . w@full -> y@shard0):
        gather the factors x and dy and rebuild dW = x^T dy on every device,
        instead of all-reducing the partial dW — whichever the cost model
        prices lower (HAP's SFB rule; cost_model.comm_time)."""
        self.sfb: dict[str, list[Instruction]] = {}
        self.sfb_done: set[str] = set()
        if self.m == 1 or self.cfg.grad_sync == "all_reduce":
            return
        uses: dict[str, list[Instruction]] = {}
        for ins in self.program.instrs:
            for d in ins.operands:
                uses.setdefault(d, []).append(ins)
        eligible = []
        for ins in self.program.instrs:
            if ins.kind != "parameter" or not self.req.get(ins.output):
                continue
            us = uses.get(ins.output, [])
            ok = bool(us) and all(u.kind == "matmul" and u.operands[1] == ins.output and u.operands[0] != ins.output
                                  and form_of_dist_id(u.operands[0]).kind == ALL_GATHER
                                  and form_of_dist_id(u.operands[0]).axis == 0
                                  and form_of_dist_id(u.output).kind == ALL_GATHER for u in us)
            if ok:
                eligible.append((ins, us))
        # weights per activation factor: one gather serves all of them (_sfb_factor)
        self._sfb_shared: dict[str, int] = {}
        for _, us in eligible:
            for x in {u.operands[0].split("@")[0] for u in us}:
                self._sfb_shared[x] = self._sfb_shared.get(x, 0) + 1
        for ins, us in eligible:
            choice = self.cfg.grad_sync if self.cfg.grad_sync != "auto" else self._price_sync(ins, us)
            self.sync_choice[ins.ref] = choice
            if choice == "sfb":
                self.sfb[ins.output] = us

    def _price_sync(self, pins: Instruction, uses: list) -> str:
        spec = self.cfg.cluster
        if spec is None:
            return "all_reduce"
        kdim, ndim = self.source_shapes[pins.ref]
        use_rows = [(u.operands[0].split("@")[0], u.ref, sum(s[0] for s in self.shapes[u.operands[0]]))
                    for u in uses]
        return price_grad_sync(spec, self.cfg.ratios, pins.ref, kdim, ndim, use_rows,
                               shared=getattr(self, "_sfb_shared", None))

    def _sfb_overlap(self) -> bool:
        g = self.group
        return bool(self.sfb) and self._side_streams() and self.cfg.overlap_sfb

    def _side_streams(self) -> bool:
        """Collectives may run on a side stream beside the compute stream
        (SFB factor gathers, bucketed gradient all-reduces): one process per
        GPU only.  Ranks sharing one GPU in one process (thread_peer_groups)
        keep every collective on their compute stream: each rank then has one
        kernel at a time within its SM cap, the caps sum to the GPU, and a
        rank's persistent GEMM can never be starved of SMs by another rank's
        peer kernel spinning for a partner that is queued behind that GEMM."""
        g = self.group
        return g.distributed and not getattr(g, "in_process", False) and (g.comm_grad is not None or g.comm is None)

    def _sfb_factor(self, did: str, bufs: dict) -> dict:
        """Row-gathered copy of an SFB factor (an activation or an output
        gradient), made once per source buffer and shared by every weight
        that uses it (both experts of a layer read the same input).  With a
        side stream the gather is issued there, ordered after the factor's
        producer by an event, and overlaps the compute stream."""
        L = self.group.local_ranks
        key = tuple(bufs[r].ptr for r in L)
        if os.environ.get("HAP_DBG_SFB_DEDUPE", "1") != "1":
            key = (did, len(self._ops), id(self._ops))
        if key in self._sfb_full:
            return self._sfb_full[key]
        rows = sum(s[0] for s in self.shapes[did])
        full = {r: self._new((rows,) + tuple(self.shapes[did][0][1:]), bufs[r].dtype) for r in L}
        if self._sfb_overlap():
            side = self._side()
            ready = self._event()
            self._keep(ready)
            self._ops.append(Op(ready.record, (self.stream,), "event.record", False))
            self._ops.append(Op(side.wait_event, (ready,), "stream.wait_event", False))
            self._emit_on = side
            try:
                self._coll_all_gather(bufs, self.shapes[did], full, 0, 0, "all_gather")
            finally:
                self._emit_on = None
        else:
            self._coll_all_gather(bufs, self.shapes[did], full, 0, 0, "all_gather")
        self._sfb_full[key] = full
        return full

    def _sfb_weight_grad(self, ins: Instruction, contrib):
        """dW = gather(x)^T . gather(dy), replicated (Id form) on every device."""
        L = self.group.local_ranks
        w = ins.operands[1]
        xdid, ydid = ins.operands[0], ins.output
        xfull = self._sfb_factor(xdid, {r: self.bufs[(xdid, r)] for r in L})
        yfull = self._sfb_factor(ydid, {r: self.grads[(ydid, r)] for r in L})
        acc = contrib(w)
        self.sfb_done.add(w)
        if self._sfb_overlap():
            self._sfb_pending.append((xfull, yfull, w, acc))
            return
        for r in L:
            self._gemm(xfull[r], True, yfull[r], False, self._grad(w, r), self.caps[r], acc)

    def _emit_sfb_pending(self):
        """The deferred SFB weight-gradient GEMMs, after one wait for the side
        stream's gathers; consecutive, so launch batching can group them."""
        if not self._sfb_pending:
            return
        done = self._event()
        self._keep(done)
        self._ops.append(Op(done.record, (self._side(),), "event.record", False))
        self._ops.append(Op(self.stream.wait_event, (done,), "stream.wait_event", False))
        for xfull, yfull, w, acc in self._sfb_pending:
            for r in self.group.local_ranks:
                self._gemm(xfull[r], True, yfull[r], False, self._grad(w, r), self.caps[r], acc)
        self._sfb_pending = []

    def _synced_params(self) -> list:
        """Parameter (and, with input_grads, placeholder) tensors realised in
        one replicated form whose gradient is all-reduced (not SFB)."""
        forms: dict = {}
        for ins in self.program.instrs:
            if ins.kind.startswith("parameter") or (self.cfg.input_grads and ins.kind.startswith("placeholder")):
                forms.setdefault(ins.ref, []).append(ins)
        return [fs[0] for fs in forms.values()
                if len(fs) == 1 and fs[0].kind in ("parameter", "placeholder") and fs[0].output not in self.sfb]

    def _flat_grads(self):
        """NCCL groups: lay the all-reduced gradients out back to back in one
        fp32 buffer, in the order the backward pass completes them, so that
        neighbouring gradients sync as one bucket (one large all-reduce runs
        at NCCL's bandwidth; dozens of small ones pay its latency each)."""
        g = self.group
        if self.m == 1 or not self._side_streams():
            return
        first_use: dict = {}
        for i, ins in enumerate(self.program.instrs):
            for d in ins.operands:
                first_use.setdefault(d, i)
        params = [f for f in self._synced_params() if self._n_contrib.get(f.output, 0) > 0]
        # a gradient is complete once the adjoint of its first consumer ran
        params.sort(key=lambda f: -first_use.get(f.output, -1))
        r = g.rank
        offs, total = [], 0
        for f in params:
            offs.append(total)
            total += (int(math.prod(self.shapes[f.output][r])) + 63) // 64 * 64   # 256-byte aligned
        if not total:
            return
        flat = torch.zeros(total, dtype=torch.float32, device=self.device)
        self._keep(flat)
        self.bytes_allocated += total * 4
        self._flat = (flat, {f.output: (o, int(math.prod(self.shapes[f.output][r]))) for f, o in zip(params, offs)})
        for f, o in zip(params, offs):
            shape = tuple(self.shapes[f.output][r])
            self.grads[(f.output, r)] = Buf(flat.narrow(0, o, max(1, int(math.prod(shape)))), F32, shape)

    def _overlap_grad_sync(self):
        """NCCL groups: all-reduce the replicated parameters' gradients on a
        side stream, bucket by bucket of the flat gradient buffer, as soon as
        the last gradient of a bucket is enqueued, so the transfers overlap
        the remaining backward kernels; the compute stream joins the side
        stream before the update."""
        g = self.group
        if self.m == 1 or not self._side_streams() or not hasattr(self, "_flat"):
            return
        flat, place = self._flat
        ready = {f.output: self._grad_ready_at[f.output] for f in self._synced_params()
                 if f.output in place and f.output in self._grad_ready_at}
        if not ready:
            return
        # buckets: runs of the flat layout of about bucket_bytes
        order = sorted(ready, key=lambda d: place[d][0])
        buckets, cur = [], []
        for d in order:
            cur.append(d)
            lo = place[cur[0]][0]
            hi = place[d][0] + place[d][1]
            if (hi - lo) * 4 >= self.cfg.bucket_bytes:
                buckets.append(cur)
                cur = []
        if cur:
            buckets.append(cur)
        self._side()
        ops = self.ops_bwd
        plan = []
        for members in buckets:
            lo = place[members[0]][0]
            hi = place[members[-1]][0] + place[members[-1]][1]
            plan.append((max(ready[d] for d in members), lo, hi, members))
        self.grad_buckets = [(hi - lo) * 4 for _, lo, hi, _ in plan]
        for pos, lo, hi, members in sorted(plan, key=lambda t: -t[0]):
            ev = self._event()
            self._keep(ev)
            ptr = flat.data_ptr() + lo * 4
            inserted = [Op(ev.record, (self.stream,), "event.record", False),
                        Op(self.comm_stream.wait_event, (ev,), "stream.wait_event", False)]
            if g.comm_grad is not None and not self._use_p2p("all_reduce", hi - lo, 4, side=True):
                inserted.append(Op(self.lib.hap_all_reduce, (g.comm_grad, ptr, ptr, hi - lo, F32,
                                                             self.comm_stream.cuda_stream), "hap_all_reduce", False))
            else:   # in place on the registered bucket, P2P kernel on the side stream
                saved, self._ops = self._ops, []
                bucket = Buf(flat.narrow(0, lo, hi - lo), F32, (hi - lo,))
                self._p2p_all_reduce(bucket, bucket, hi - lo, stream_ptr=self.comm_stream.cuda_stream)
                inserted += self._ops
                self._ops = saved
            ops[pos:pos] = inserted
            self.overlapped.update(members)
        done = self._event()
        self._keep(done)
        ops.append(Op(done.record, (self.comm_stream,), "event.record", False))
        ops.append(Op(self.stream.wait_event, (done,), "stream.wait_event", False))

    def _finish_update(self, written: set):
        """Turn per-device parameter gradients into true gradients and apply SGD.

        Replicated (@full) parameter gradients are partial sums: all-reduced,
        unless SFB already produced them replicated.  Sharded gradients are
        already the device's slice of the true gradient."""
        L = self.group.local_ranks
        sfb_done = self.sfb_done
        self.param_grads: dict[tuple[str, int], Buf] = {}
        forms: dict[str, list[Instruction]] = {}
        for ins in self.program.instrs:
            if ins.kind.startswith("parameter") or (self.cfg.input_grads and ins.kind.startswith("placeholder")):
                forms.setdefault(ins.ref, []).append(ins)
        for ref, fs in forms.items():
            live = [f for f in fs if f.output in written]
            if not live:
                continue
            if len(fs) == 1:
                f = fs[0]
                g = {r: self.grads[(f.output, r)] for r in L}
                if (f.kind in ("parameter", "placeholder") and f.output not in sfb_done and self.m > 1
                        and f.output not in self.overlapped):
                    self._coll_all_reduce(g, g, 0)
                for r in L:
                    self.param_grads[(f.output, r)] = g[r]
            else:
                # A parameter realised in several forms: assemble the full
                # gradient (partial form), all-reduce it, hand each form its part.
                full_shape = self.source_shapes[ref]
                fullg = {r: self._new(full_shape, F32) for r in L}
                first = True
                for f in live:
                    for r in L:
                        g = self.grads[(f.output, r)]
                        if f.kind.endswith("_shard"):
                            sizes = self._sizes(ref, f.axis)
                            o = offsets(sizes)[r]
                            if first:
                                self._emit("hap_fill", fullg[r].ptr, F32, 0.0, fullg[r].numel, self._sptr())
                            self._block(g, _view(g.shape, f.axis), 0, fullg[r], _view(full_shape, f.axis), o,
                                        g.shape[f.axis], self.caps[r], 1)
                        else:
                            scale = 1.0 / self.m if f.output in sfb_done else 1.0
                            self._copy(g, fullg[r], self.caps[r], accumulate=int(not first), alpha=scale)
                    first = False
                if self.m > 1:
                    self._coll_all_reduce(fullg, fullg, 0)
                for f in fs:
                    for r in L:
                        if f.kind.endswith("_shard"):
                            sizes = self._sizes(ref, f.axis)
                            part = self._new(self.shapes[f.output][r], F32)
                            self._block(fullg[r], _view(full_shape, f.axis), offsets(sizes)[r], part,
                                        _view(part.shape, f.axis), 0, sizes[r], self.caps[r])
                            self.param_grads[(f.output, r)] = part
                        else:
                            self.param_grads[(f.output, r)] = fullg[r]
        self._ops = self.ops_upd = []
        if self.cfg.lr:
            self._compile_sgd()

    def _compile_sgd(self):
        """One multi-tensor SGD launch per local device and weight dtype: a
        device table of {master, grad, weight, n, first_chunk} records."""
        groups: dict = {}
        for (did, r), g in self.param_grads.items():
            if (did, r) not in self.masters:
                continue
            mst, wb = self.masters[(did, r)], self.bufs[(did, r)]
            groups.setdefault((r, wb.dtype), []).append((mst, g, wb))
        self._sgd_items = groups
        for (r, wdt), items in sorted(groups.items()):
            self._emit_sgd(items, r, wdt, self._sptr())

    def _emit_sgd(self, items, r, wdt, stream_ptr):
        import struct

        records, chunk = bytearray(), 0
        for mst, g, wb in items:
            records += struct.pack("<QQQqq", mst.ptr, g.ptr, wb.ptr, mst.numel, chunk)
            chunk += (mst.numel + 8191) // 8192
        table = torch.frombuffer(records, dtype=torch.uint8).to(self.device)
        self._keep(table)
        self._emit("hap_sgd_multi", table.data_ptr(), len(items), chunk, wdt, float(self.cfg.lr),
                   self.caps[r], stream_ptr)

    def _want_sgd_overlap(self) -> bool:
        """cfg.sgd_overlap "auto": overlap when the update's HBM time (14 B per
        parameter) exceeds a quarter of the backward GEMMs' tensor time — the
        regime where those GEMMs are small and leave SMs and HBM idle
        (BERT-MoE: 1.6 GB of update against 114 GFLOP; BERT: 1.2 GB against
        2.8 TFLOP, where the GEMMs fill every SM and the update only contends)."""
        mode = str(self.cfg.sgd_overlap)
        if mode in ("0", "1"):
            return mode == "1"
        params = sum(it[0].numel for items in self._sgd_items.values() for it in items)
        flops = sum(2 * m["M"] * m["N"] * m["K"] for op in self.ops_bwd if op.gemm is not None
                    for m in op.gemm.get("members", [op.gemm]))
        return params * 14 / 6.5e12 > 0.25 * flops / 1.4e15

    def _overlap_sgd(self):
        """Move the SGD update into the backward, on a side stream.  For each
        parameter, its ready point is the last backward op that touches its
        gradient, fp32 master or bf16 weight (GEMMs by their descriptors,
        direct-pointer kernels by their pointer arguments).  Parameters are
        updated in groups of about one layer (>= 1/12 of all parameters) right
        after the group's last ready point: fork (event on the compute stream),
        hap_sgd_multi on the side stream, one join at the end of the step.
        Only when every backward op is analysable (no collectives: m = 1 per
        process); otherwise the single update at the end stays."""
        if any(op.gemm is None and op.what not in self._DIRECT_OPS for op in self.ops_bwd):
            return
        if len(self._sgd_items) != 1:
            return
        ((r, wdt), items), = self._sgd_items.items()

        def span(b):
            return (b.ptr, b.ptr + max(1, b.numel) * (4 if b.dtype == F32 else 2))

        def touches(op, ranges):
            if op.gemm is not None:
                rd, wr = self._gemm_ranges(op.gemm)
                return any(lo < hi2 and lo2 < hi for lo, hi in rd + wr for lo2, hi2 in ranges)
            return any(isinstance(a, int) and any(lo <= a < hi for lo, hi in ranges) for a in op.args)

        ready = []
        for it in items:
            ranges = [span(b) for b in it]
            last = -1
            for i, op in enumerate(self.ops_bwd):
                if touches(op, ranges):
                    last = i
            ready.append(last)
        order = sorted(range(len(items)), key=lambda j: ready[j])
        total = sum(it[0].numel for it in items)
        side = self._stream()
        self.sgd_stream = side
        groups, cur, size = [], [], 0
        for j in order:
            cur.append(j)
            size += items[j][0].numel
            if size * 12 >= total:
                groups.append(cur)
                cur, size = [], 0
        if cur:
            groups.append(cur)
        inserts: dict = {}
        saved = self._ops
        for grp in groups:
            at = max(ready[j] for j in grp)
            self._ops = []
            ev = self._event()
            self._keep(ev)
            self._ops.append(Op(ev.record, (self.stream,), "event.record", False))
            self._ops.append(Op(side.wait_event, (ev,), "stream.wait_event", False))
            self._emit_sgd([items[j] for j in grp], r, wdt, side.cuda_stream)
            inserts.setdefault(at, []).extend(self._ops)
        self._ops = saved
        out = list(inserts.get(-1, []))
        for i, op in enumerate(self.ops_bwd):
            out.append(op)
            out.extend(inserts.get(i, []))
        done = self._event()
        self._keep(done)
        out.append(Op(done.record, (side,), "event.record", False))
        out.append(Op(self.stream.wait_event, (done,), "stream.wait_event", False))
        self.ops_bwd[:] = out
        self.ops_upd[:] = []
        self.sgd_stats = (len(groups), len(items))

    # ------------------------------------------------------------------ binding
    def load(self, inputs: dict):
        """Bind every source (interpreter.py:132-138): float64 host arrays ->
        device working copies (+ fp32 masters for parameters), sliced per the
        shard table."""
        self.stream.synchronize()
        for ins in self.program.instrs:
            if ins.kind not in SOURCE_KINDS:
                continue
            try:
                value = np.asarray(inputs[ins.ref], dtype=np.float64)
            except KeyError:
                raise ExecutionError(f"no binding for source tensor {ins.ref!r}") from None
            if tuple(value.shape) != self.source_shapes[ins.ref]:
                raise ExecutionError(f"binding for {ins.ref!r} has shape {value.shape}, "
                                     f"want {self.source_shapes[ins.ref]}")
            full = torch.from_numpy(np.ascontiguousarray(value, dtype=np.float32))
            for r in self.group.local_ranks:
                if ins.kind.endswith("_shard"):
                    sizes = self._sizes(ins.ref, ins.axis)
                    o = offsets(sizes)
                    part = full.narrow(ins.axis, o[r], sizes[r]).contiguous()
                else:
                    part = full
                buf = self.bufs[(ins.output, r)]
                buf.tensor[:part.numel()].copy_(part.reshape(-1).to(self.device), non_blocking=False)
                if (ins.output, r) in self.masters:
                    self.masters[(ins.output, r)].tensor[:part.numel()].copy_(part.reshape(-1).to(self.device))
        # the copies ran on torch's current stream, which the executor's own
        # (non-blocking) stream does not wait for: done before the next step
        if not self.dry:
            torch.cuda.current_stream(self.device).synchronize()

    def source_buffers(self, ref: str) -> dict[int, tuple[Instruction, Buf]]:
        out = {}
        for ins in self.program.instrs:
            if ins.kind in SOURCE_KINDS and ins.ref == ref:
                for r in self.group.local_ranks:
                    out.setdefault(r, []).append((ins, self.bufs[(ins.output, r)]))
        return out

    # ------------------------------------------------------------------ running
    def _run(self, ops: list[Op]):
        for op in ops:
            st = op.fn(*op.args)
            if st:
                check(st, op.what)

    def forward(self):
        with torch.cuda.stream(self.stream):
            self._run(self.ops_fwd)

    def backward(self):
        with torch.cuda.stream(self.stream):
            self._run(self.ops_bwd)
            self._run(self.ops_upd)

    def step(self):
        """One training iteration: forward, backward, gradient sync, update."""
        if self.graph is not None:
            with torch.cuda.stream(self.stream):
                self.graph.replay()
            return
        with torch.cuda.stream(self.stream):
            self._run(self.ops_fwd)
            self._run(self.ops_bwd)
            self._run(self.ops_upd)

    def capture(self, warmup: bool = True):
        """Record forward+backward+update into one CUDA graph (all ops were
        compiled against self.stream, the capture stream).  ``warmup``: one
        eager step first (kernel attributes, NCCL setup, per-stream
        workspaces).  Ranks that live in one process (thread_peer_groups) warm
        up together (their peer kernels wait for each other) and then capture
        one after another with warmup=False: torch's graph capture frees cached
        memory on entry, which would invalidate another thread's capture."""
        if warmup:
            self.step()
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        # thread-local capture: NCCL's proxy thread keeps issuing CUDA calls
        # while this thread captures the collectives' kernels.
        with torch.cuda.graph(g, stream=self.stream, capture_error_mode="thread_local"):
            self._run(self.ops_fwd)
            self._run(self.ops_bwd)
            self._run(self.ops_upd)
        self.graph = g
        return g

    _COLLECTIVE_OPS = ("hap_all_reduce", "hap_all_gather_v", "hap_grouped_broadcast", "hap_reduce_scatter_v",
                       "hap_all_to_all_v", "hap_p2p_all_gather_push", "hap_p2p_all_gather_v",
                       "hap_p2p_reduce_scatter_direct", "hap_p2p_reduce_scatter_v", "hap_p2p_all_reduce",
                       "hap_p2p_all_to_all")

    def collective_impls(self) -> dict:
        """Collective launches per step by implementation (NCCL calls vs the
        NVLink peer-memory kernels)."""
        out: dict = {}
        for op in self.ops_fwd + self.ops_bwd + self.ops_upd:
            if op.what in self._COLLECTIVE_OPS:
                out[op.what] = out.get(op.what, 0) + 1
        return dict(sorted(out.items()))

    def kernel_launches(self, phase: str = "step") -> int:
        ops = {"forward": self.ops_fwd, "backward": self.ops_bwd + self.ops_upd,
               "step": self.ops_fwd + self.ops_bwd + self.ops_upd}[phase]
        return sum(1 for op in ops if op.kernel)

    def losses(self) -> list[float]:
        """Per-device loss values of the last forward (host sync)."""
        self.stream.synchronize()
        vals = {r: float(self.loss_buf[r].tensor[0].item()) for r in self.group.local_ranks}
        if self.group.distributed:
            return [float(v) for v in self.group.exchange(vals[self.group.rank])]
        return [vals[r] for r in range(self.m)]

    def tensor(self, did: str, r: int) -> torch.Tensor:
        b = self.bufs[(did, r)]
        return b.tensor[:b.numel].view(b.shape) if b.shape else b.tensor[:1].view(())

    def gradient(self, ref: str) -> dict[int, tuple[Instruction, torch.Tensor]]:
        """Synchronised gradient of source ``ref`` per local device/form."""
        out = {}
        for (did, r), g in self.param_grads.items():
            if did.rpartition("@")[0] == ref:
                out.setdefault(r, []).append((did, g.tensor[:g.numel].view(g.shape)))
        return out

    def close(self):
        if getattr(self, "_symm", None):
            torch.cuda.synchronize(self.device)
            for ctx in self._symm.values():
                check(self.lib.hap_symm_destroy(ctx), "hap_symm_destroy")
            self._symm = {}
        if self.__dict__.get("_own_streams"):
            self.graph = None
            torch.cuda.synchronize(self.device)
            dev = self.device.index if self.device.index is not None else torch.cuda.current_device()
            _release_streams(dev, self._own_streams)
        if self.group is not None:
            self.group.close()
