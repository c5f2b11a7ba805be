"""Shared case list and checks of the multi-device parity runs
(tests/multi/nccl_parity.py: one process per GPU over NCCL;
tests/multi/peer_ranks.py: ranks as threads of one process on one GPU, NVLink
peer-memory kernels only).  Losses are checked against the oracle evaluated in
the executor's storage precision — rtol 5e-3 in bf16, 1e-3 in fp32 — relative
to max(|loss|, 1) as the reference's check_equivalence scales
(interpreter.py:264-277); gradients against the oracle's distributed adjoint
in storage precision at the north_star rtol (2e-2 bf16, 1e-3 fp32) of the
largest reference magnitude."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

import goldens  # noqa: E402
from oracle import interpreter_np as O  # noqa: E402

LOSS_RTOL = {"bf16": 5e-3, "fp32": 1e-3}
GRAD_RTOL = {"bf16": 2e-2, "fp32": 1e-3}


def cases(world: int) -> list:
    """(name, plan document, graph name, inputs) of every golden program for
    ``world`` devices: the reference planner's plans and the enumerated
    programs with collectives."""
    out = []
    for gname, cname in goldens.value_cases():
        doc = goldens.plan(gname, cname)
        if doc["devices"] == world:
            vals = goldens.values(gname, cname)
            out.append((f"{gname}.{cname}", doc, gname, goldens.inputs(goldens.graph(gname), vals, goldens.seeds(vals)[0])))
    for stem in goldens.program_cases():
        doc, vals, gname = goldens.program_case(stem)
        if doc["devices"] == world:
            inputs = {k.split(":", 2)[2]: vals[k] for k in vals.files if k.startswith("seed0:input:")}
            out.append((stem, doc, gname, inputs))
    return out


def check(label: str, doc: dict, gname: str, inputs: dict, dtype: str, losses: list, grads: dict) -> list:
    """Failures (strings) of one run.  ``grads``: ref -> {rank: [(did, array)]}."""
    g = goldens.graph(gname)
    program, m, table = O.load_plan(doc)
    _, want = O.run_distributed(program, m, inputs, table, precision=dtype)
    _, sg, _ = O.train_step(program, m, inputs, table, {n.id: n.shape for n in g.nodes}, precision=dtype)
    failures = []
    for got, w in zip(losses, want):
        if abs(got - float(w)) > LOSS_RTOL[dtype] * max(1.0, abs(float(w))):
            failures.append(f"{label}: losses {losses} vs {[float(v) for v in want]}")
            break
    for ref, value in sg.items():
        per = grads.get(ref, {})
        if not per:
            failures.append(f"{label}: no gradient for {ref}")
            continue
        for r, forms in per.items():
            for did, grad in forms:
                if "@shard" in did:
                    axis = int(did.rsplit("shard", 1)[1])
                    sizes = table[(ref, axis)]
                    off = int(np.sum(sizes[:r]))
                    value_r = np.take(value, np.arange(off, off + sizes[r]), axis=axis)
                else:
                    value_r = value
                if value_r.size == 0:
                    continue
                err = float(np.max(np.abs(grad - value_r))) / max(float(np.max(np.abs(value))), 1e-3)
                if err > GRAD_RTOL[dtype]:
                    failures.append(f"{label}: grad {did}@{r} rel err {err:.3g}")
    return failures
