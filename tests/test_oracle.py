"""The CPU oracle is pinned to the reference: its forward execution must
reproduce the reference interpreter's outputs on the golden cases, its
single-device gradients the reference's central differences, and its
distributed adjoint the single-device gradients."""
import numpy as np
import pytest

import goldens
from oracle import interpreter_np as O

CASES = goldens.value_cases()


@pytest.mark.parametrize("gname,cname", CASES)
def test_oracle_forward_matches_reference_interpreter(gname, cname):
    g = goldens.graph(gname)
    vals = goldens.values(gname, cname)
    program, m, table = O.load_plan(goldens.plan(gname, cname))
    for seed in goldens.seeds(vals):
        inputs = goldens.inputs(g, vals, seed)
        env, losses = O.run_distributed(program, m, inputs, table)
        want = vals[f"seed{seed}:losses"]
        got = np.array([float(v) for v in losses])
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
        single = float(O.eval_single(g, inputs)[g.loss])
        assert abs(single - float(vals[f"seed{seed}:single"])) <= 1e-12 * max(1.0, abs(single))
        if seed == goldens.seeds(vals)[0]:
            for did, insts in goldens.env(vals).items():
                assert len(env[did]) == m
                for dev, ref in enumerate(insts):
                    np.testing.assert_allclose(env[did][dev], ref, rtol=1e-12, atol=1e-12,
                                               err_msg=f"{did} device {dev}")


GRAD_GRAPHS = sorted({g for g, _ in CASES if not g.startswith(("mlp", "bert", "moe", "vitmoe"))})


@pytest.mark.parametrize("gname", GRAD_GRAPHS)
def test_oracle_gradient_matches_reference_finite_differences(gname):
    g = goldens.graph(gname)
    fd = np.load(f"{goldens.GOLDEN}/grads/{gname}.npz")
    inputs = {k[6:]: fd[k] for k in fd.files if k.startswith("input:")}
    grads = O.grad_single(g, inputs)
    for name, value in grads.items():
        want = fd[f"grad:{name}"]
        scale = max(1.0, float(np.max(np.abs(want))))
        # relu kinks make central differences exact only away from 0; inputs are
        # standard normal so no element sits within eps of a kink.
        assert np.max(np.abs(value - want)) <= 1e-5 * scale, name


@pytest.mark.parametrize("gname,cname", CASES)
def test_distributed_adjoint_matches_single_device_gradient(gname, cname):
    g = goldens.graph(gname)
    vals = goldens.values(gname, cname)
    program, m, table = O.load_plan(goldens.plan(gname, cname))
    seed = goldens.seeds(vals)[0]
    inputs = goldens.inputs(g, vals, seed)
    shapes = {n.id: n.shape for n in g.nodes}
    _, sgrads, _ = O.train_step(program, m, inputs, table, shapes)
    want = O.grad_single(g, inputs)
    for name, value in want.items():
        scale = max(1.0, float(np.max(np.abs(value))))
        assert np.max(np.abs(sgrads[name] - value)) <= 1e-9 * scale, name
