"""Executor parity on the B200: the CUDA path (through the C ABI) against the
reference interpreter's golden outputs and the CPU oracle, for every golden
plan and every enumerated program with collectives, with all m program
devices emulated on one GPU (LocalGroup).  Tolerances: rtol 2e-2 in bf16,
1e-3 in fp32 (north_star), relative to max(|reference|, 1) per value and to
the largest reference magnitude for gradient tensors; bf16 losses also
within 5e-3 of the oracle evaluated in bf16 storage precision."""
import numpy as np
import pytest
import torch

import goldens
from oracle import interpreter_np as O
from paper_2401_05965_b200.executor import ExecConfig, Executor, LocalGroup
from paper_2401_05965_b200.program import DistributedProgram
from paper_2401_05965_b200.sharding import table_from_plan

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

RTOL = {"bf16": 2e-2, "fp32": 1e-3}


def _run(doc, g, inputs, dtype, lr=0.0, grad_sync="auto"):
    prog = DistributedProgram.from_json(doc["program"])
    m = int(doc["devices"])
    shapes = {n.id: n.shape for n in g.nodes if n.op in ("Placeholder", "Parameter")}
    ex = Executor(prog, m, table_from_plan(doc), shapes, group=LocalGroup(m),
                  config=ExecConfig(dtype=dtype, lr=lr, input_grads=True, grad_sync=grad_sync))
    ex.load(inputs)
    ex.step()
    torch.cuda.synchronize()
    return ex


# bf16 storage alone moves these losses more than the bf16 tolerance away
# from the float64 reference: the oracle run in bf16 storage precision is
# itself that far off (asserted below), so the executor is held to the
# storage-precision oracle for them.  mlp.ratio12 (configs[0]) sums 65 536
# terms of |.|-sum 3.7e4 to a loss of 42: 3.8 % in bf16 storage.
KNOWN_BF16_STORAGE_GAP = {"mlp.ratio12"}
LOSS_RTOL_STORAGE = 5e-3    # bf16 run vs the oracle in bf16 storage precision


def _check_losses(ex, doc, inputs, want, dtype, case):
    """Losses against (1) the float64 reference goldens at the north_star
    tolerance, relative to max(|loss|, 1) as the reference's check_equivalence
    scales (interpreter.py:264-277), and (2) in bf16, the oracle evaluated in
    the executor's storage precision at 5e-3."""
    got = np.array(ex.losses())
    scale = np.maximum(np.abs(want), 1.0)
    if dtype == "bf16":
        program, m, table = O.load_plan(doc)
        _, stored = O.run_distributed(program, m, inputs, table, precision="bf16")
        stored = np.array(stored, dtype=np.float64)
        assert np.all(np.abs(got - stored) <= LOSS_RTOL_STORAGE * np.maximum(np.abs(stored), 1.0)), (got, stored)
        if case in KNOWN_BF16_STORAGE_GAP:
            assert np.any(np.abs(stored - want) > RTOL[dtype] * scale), f"{case} no longer needs the exception"
            return
    assert np.all(np.abs(got - want) <= RTOL[dtype] * scale), (got, want)


def _check_grads(ex, g, inputs, dtype, doc):
    """Gradients against the oracle's distributed adjoint run in the
    executor's storage precision (interpreter_np.storage_dtypes): float64
    arithmetic, values rounded to bf16/fp32 exactly where the device stores
    them.  Against pure float64, a ReLU input within one bf16 ulp of zero
    flips its mask (chain4: activations ~600), which no bf16 run can match."""
    program, m, table = O.load_plan(doc)
    shapes = {n.id: n.shape for n in g.nodes}
    _, want, _ = O.train_step(program, m, inputs, table, shapes, precision=dtype)
    for ref, value in want.items():
        per = ex.gradient(ref)
        assert per, f"no gradient for {ref}"
        for r, forms in per.items():
            for did, grad in forms:
                grad = grad.float().cpu().numpy().astype(np.float64)
                if "@shard" in did:
                    axis = int(did.rsplit("shard", 1)[1])
                    sizes = ex._sizes(ref, axis)
                    off = int(np.sum(sizes[:r]))
                    expect = np.take(value, np.arange(off, off + sizes[r]), axis=axis)
                else:
                    expect = value
                scale = max(float(np.max(np.abs(value))), 1e-3)
                err = float(np.max(np.abs(grad - expect))) / scale if grad.size else 0.0
                assert err <= RTOL[dtype], f"{did} device {r}: rel err {err}"


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("gname,cname", goldens.value_cases())
def test_planned_programs_match_reference(gname, cname, dtype):
    g = goldens.graph(gname)
    vals = goldens.values(gname, cname)
    doc = goldens.plan(gname, cname)
    seed = goldens.seeds(vals)[0]
    inputs = goldens.inputs(g, vals, seed)
    ex = _run(doc, g, inputs, dtype)
    want = vals[f"seed{seed}:losses"]
    _check_losses(ex, doc, inputs, want, dtype, f"{gname}.{cname}")
    for did, insts in goldens.env(vals).items():
        for r, want in enumerate(insts):
            got = ex.tensor(did, r).float().cpu().numpy()
            scale = max(float(np.max(np.abs(want))) if want.size else 1.0, 1.0)
            assert got.shape == want.shape
            assert (np.max(np.abs(got - want)) if want.size else 0.0) <= RTOL[dtype] * scale, did
    _check_grads(ex, g, inputs, dtype, doc)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("stem", goldens.program_cases())
def test_programs_with_collectives_match_reference(stem, dtype):
    doc, vals, gname = goldens.program_case(stem)
    g = goldens.graph(gname)
    inputs = {k.split(":", 2)[2]: vals[k] for k in vals.files if k.startswith("seed0:input:")}
    ex = _run(doc, g, inputs, dtype)
    want = vals["seed0:losses"]
    _check_losses(ex, doc, inputs, want, dtype, stem)
    _check_grads(ex, g, inputs, dtype, doc)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("case", ["moe2_b2.b200x2", "moe2_b2.b200x4", "mlp.ratio12"])
def test_sufficient_factor_broadcasting_matches_reference(case, dtype):
    """Every replicated weight rebuilt from gathered factors (x, dy) gives the
    reference gradient, as the all-reduce path does."""
    gname, cname = case.split(".")
    g = goldens.graph(gname)
    vals = goldens.values(gname, cname)
    doc = goldens.plan(gname, cname)
    inputs = goldens.inputs(g, vals, goldens.seeds(vals)[0])
    ex = _run(doc, g, inputs, dtype, grad_sync="sfb")
    assert ex.sync_choice and set(ex.sync_choice.values()) == {"sfb"}, ex.sync_choice
    assert ex.sfb_done == set(ex.sfb)
    _check_grads(ex, g, inputs, dtype, doc)


def test_sgd_update_matches_oracle():
    g = goldens.graph("chain4")
    doc = goldens.plan("chain4", "hetero2")
    vals = goldens.values("chain4", "hetero2")
    inputs = goldens.inputs(g, vals, 0)
    ex = _run(doc, g, inputs, "fp32", lr=0.01)
    program, m, table = O.load_plan(doc)
    shapes = {n.id: n.shape for n in g.nodes}
    _, _, updated = O.train_step(program, m, inputs, table, shapes, lr=0.01)
    for ref, want in updated.items():
        for (did, r), master in ex.masters.items():
            if did.rpartition("@")[0] != ref:
                continue
            got = master.tensor[:master.numel].view(master.shape).cpu().numpy()
            if "@shard" in did:
                axis = int(did.rsplit("shard", 1)[1])
                sizes = ex._sizes(ref, axis)
                off = int(np.sum(sizes[:r]))
                want_r = np.take(want, np.arange(off, off + sizes[r]), axis=axis)
            else:
                want_r = want
            assert np.max(np.abs(got - want_r)) <= 1e-4 * max(1.0, np.max(np.abs(want_r)))


def test_cuda_graph_replay_matches_eager():
    """One captured step replays exactly what the eager op list computes."""
    g = goldens.graph("bert2_b2")
    doc = goldens.plan("bert2_b2", "b200x2")
    vals = goldens.values("bert2_b2", "b200x2")
    inputs = goldens.inputs(g, vals, 0)
    prog = DistributedProgram.from_json(doc["program"])
    shapes = {n.id: n.shape for n in g.sources()}
    ex = Executor(prog, 2, table_from_plan(doc), shapes, group=LocalGroup(2),
                  config=ExecConfig(dtype="bf16", lr=1e-7, sm_caps=[148, 104]))
    ex.load(inputs)
    ex.step()
    eager_loss = ex.losses()
    eager = {k: b.tensor.float().cpu().clone() for k, b in ex.masters.items()}
    ex.capture()
    ex.load(inputs)
    ex.step()
    graph_loss = ex.losses()
    assert np.allclose(eager_loss, graph_loss, rtol=1e-5), (eager_loss, graph_loss)
    for k, b in ex.masters.items():
        assert torch.allclose(b.tensor.float().cpu(), eager[k], rtol=1e-5, atol=1e-6), k
    for _ in range(5):
        ex.step()
    assert all(np.isfinite(ex.losses()))


@pytest.mark.parametrize("workload", ["bert", "moe"])
def test_fused_epilogues_match_unfused(workload):
    """The executor with GEMM-epilogue fusion (swish after f1, residual adds,
    deferred residual-gradient copies, the swish adjoint after the dg GEMM)
    against the same program with every elementwise op as its own kernel:
    fewer launches, same losses and gradients (bf16 rounding points are the
    same, so only fp32 contraction differences remain)."""
    from paper_2401_05965_b200 import api, workloads

    g = workloads.bert(layers=2, batch=8, seq=128) if workload == "bert" else \
        workloads.moe_stack(layers=2, batch=8, seq=128)
    inputs = workloads.synthetic_inputs(g, 3, scaled=True)
    shapes = {n.id: n.shape for n in g.sources()}
    out = {}
    for fuse in (False, True):
        ex = Executor(api.single_device_program(g), 1, {}, shapes, group=LocalGroup(1),
                      config=ExecConfig(dtype="bf16", fuse_epilogue=fuse, fuse_swish_fwd=fuse))
        ex.load(inputs)
        ex.step()
        torch.cuda.synchronize()
        grads = {}
        for ref in ("l0_W1", "l1_W2", "l0_Wq") if workload == "bert" else ("l0_e0_W1", "l1_e1_W2"):
            for _, forms in ex.gradient(ref).items():
                grads[ref] = forms[0][1].float().cpu()
        out[fuse] = (ex.losses()[0], grads, ex.kernel_launches())
        ex.close()
    (l0, g0, k0), (l1, g1, k1) = out[False], out[True]
    assert k1 < k0, (k0, k1)
    assert abs(l1 - l0) <= 1e-3 * max(1.0, abs(l0)), (l0, l1)
    for ref in g0:
        err = float((g1[ref] - g0[ref]).abs().max() / g0[ref].abs().max())
        assert err < 1e-2, (ref, err)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_sgd_overlap_matches_single_update(dtype):
    """The SGD update moved into the backward on a side stream (one launch
    per parameter group right after the backward's last touch of the group)
    computes what the single update at the end computes: two steps, eager and
    graph-replayed, same masters and losses."""
    from paper_2401_05965_b200 import api, workloads

    g = workloads.moe_stack(layers=2, batch=2, seq=128)
    inputs = workloads.synthetic_inputs(g, 5, scaled=True)
    shapes = {n.id: n.shape for n in g.sources()}
    out = {}
    for overlap in ("0", "1"):
        ex = Executor(api.single_device_program(g), 1, {}, shapes, group=LocalGroup(1),
                      config=ExecConfig(dtype=dtype, lr=1e-4, sgd_overlap=overlap))
        assert (ex.sgd_stats[0] > 1) == (overlap == "1"), ex.sgd_stats
        ex.load(inputs)
        ex.step()
        ex.step()
        eager = (ex.losses(), {k: b.tensor.float().cpu().clone() for k, b in ex.masters.items()})
        ex.capture()
        ex.load(inputs)
        ex.step()
        ex.step()
        graph = (ex.losses(), {k: b.tensor.float().cpu().clone() for k, b in ex.masters.items()})
        out[overlap] = (eager, graph)
        ex.close()
    tol = 1e-6 if dtype == "fp32" else 1e-4
    for (l0, m0), (l1, m1) in zip(out["0"], out["1"]):
        assert np.allclose(l0, l1, rtol=tol, atol=0), (l0, l1)
        for k in m0:
            assert torch.allclose(m0[k], m1[k], rtol=tol, atol=0), k
