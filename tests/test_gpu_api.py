"""The reference-facing entry points on the B200 (paper_2401_05965_b200.api
mirrors interpreter.py:217-277; cli mirrors cli.py:131-172): run_distributed
with its executor cache and debug form check, run_single, check_equivalence,
and the `verify` / `run` commands."""
import os

import numpy as np
import pytest
import torch

import goldens
from oracle import interpreter_np as O
from paper_2401_05965_b200 import api, executor
from paper_2401_05965_b200.cli import main as cli_main
from paper_2401_05965_b200.executor import ExecutionError
from paper_2401_05965_b200.program import DistributedProgram, Instruction
from paper_2401_05965_b200.sharding import table_from_plan

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

CASES = ["chain4.hetero2", "matmul_unary.skew2", "skip_connection.homog3", "bert2_b2.b200x2", "mlp.ratio12"]


def _case(case):
    gname, cname = case.split(".")
    g = goldens.graph(gname)
    doc = goldens.plan(gname, cname)
    vals = goldens.values(gname, cname)
    return g, doc, goldens.inputs(g, vals, goldens.seeds(vals)[0]), vals


@pytest.mark.parametrize("case", CASES)
def test_run_distributed_matches_reference_and_reuses_the_executor(case, monkeypatch):
    g, doc, inputs, vals = _case(case)
    prog = DistributedProgram.from_json(doc["program"])
    table = table_from_plan(doc)
    builds = []
    real = executor.Executor.__init__

    def counting(self, *a, **k):
        builds.append(1)
        real(self, *a, **k)

    monkeypatch.setattr(executor.Executor, "__init__", counting)
    api.clear_cache()
    first = api.run_distributed(prog, doc["devices"], inputs, table, dtype="fp32")
    second = api.run_distributed(prog, doc["devices"], inputs, table, dtype="fp32")
    assert len(builds) == 1, "the second call must reuse the compiled executor"
    assert [float(v) for v in first] == [float(v) for v in second]
    want = vals[f"seed{goldens.seeds(vals)[0]}:losses"]
    assert np.all(np.abs(np.array(first) - want) <= 1e-3 * np.maximum(np.abs(want), 1.0))


@pytest.mark.parametrize("case", CASES)
def test_debug_mode_checks_every_declared_form(case):
    g, doc, inputs, _ = _case(case)
    prog = DistributedProgram.from_json(doc["program"])
    reference = O.eval_single(g, inputs)
    api.run_distributed(prog, doc["devices"], inputs, table_from_plan(doc), debug=True, reference=reference,
                        dtype="fp32")
    with pytest.raises(AssertionError, match="needs reference"):
        api.run_distributed(prog, doc["devices"], inputs, table_from_plan(doc), debug=True, dtype="fp32")


def test_debug_mode_catches_a_violated_form():
    """A realised tensor that does not match its declared form (here: the
    reference value of one row-sharded matmul output shifted) is rejected, as
    the reference's check_form rejects it."""
    g, doc, inputs, _ = _case("bert2_b2.b200x2")
    prog = DistributedProgram.from_json(doc["program"])
    target = next(ins for ins in prog.instrs if ins.kind == "matmul" and ins.output.endswith("@shard0"))
    reference = dict(O.eval_single(g, inputs))
    reference[target.ref] = np.asarray(reference[target.ref]) + 1.0
    with pytest.raises(ExecutionError, match="violates its declared property"):
        api.run_distributed(prog, doc["devices"], inputs, table_from_plan(doc), debug=True, reference=reference,
                            dtype="fp32")


@pytest.mark.parametrize("case", CASES)
def test_run_single_matches_oracle(case):
    g, _, inputs, _ = _case(case)
    want = float(O.eval_single(g, inputs)[g.loss])
    got = float(api.run_single(g, inputs))
    assert abs(got - want) <= 1e-3 * max(abs(want), 1.0), (got, want)


@pytest.mark.parametrize("case,dtype", [(c, "fp32") for c in CASES] + [("chain4.hetero2", "bf16")])
def test_check_equivalence_passes_for_planned_programs(case, dtype):
    g, doc, _, _ = _case(case)
    prog = DistributedProgram.from_json(doc["program"])
    rep = api.check_equivalence(g, prog, doc["devices"], table_from_plan(doc), trials=2, dtype=dtype)
    assert rep.passed, rep


def test_check_equivalence_rejects_a_wrong_program():
    """A program whose attention gate applies tanh where the graph has a
    sigmoid computes a different loss: the equivalence check reports it."""
    g, doc, _, _ = _case("bert2_b2.b200x2")
    prog = DistributedProgram.from_json(doc["program"])
    instrs = []
    for ins in prog.instrs:
        if ins.kind == "elemwise_unary" and ins.ref == "l0_att":
            ins = Instruction(ins.kind, ins.ref, operands=ins.operands, output=ins.output, tag="tanh")
        instrs.append(ins)
    wrong = DistributedProgram(instrs=tuple(instrs), loss=prog.loss)
    rep = api.check_equivalence(g, wrong, doc["devices"], table_from_plan(doc), trials=1, dtype="fp32")
    assert not rep.passed and rep.max_rel_err > 1e-3, rep


def test_cli_verify_and_run(capsys):
    plan = os.path.join(goldens.GOLDEN, "plans", "chain4.hetero2.json")
    graph = os.path.join(goldens.GOLDEN, "graphs", "chain4.json")
    cluster = os.path.join(goldens.GOLDEN, "clusters", "hetero2.json")
    assert cli_main(["verify", plan, graph, cluster, "--trials", "2"]) == 0
    out = capsys.readouterr().out
    assert "estimate: ok" in out and "shard_table: ok" in out and "equivalence: 2 trials" in out
    assert cli_main(["run", plan, graph, "--steps", "2", "--lr", "0.001", "--dtype", "bf16"]) == 0
    out = capsys.readouterr().out
    assert "step 1: losses" in out
