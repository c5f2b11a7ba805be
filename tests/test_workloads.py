"""The bench workloads' programs are the ones the HAP planner emits.

bench.py's N = 1 line runs the program of the N = 2 golden plan re-targeted
to one device (workloads.planned_program), because the planner's m = 1 search
does not finish for 12 layers.  That is sound because the planner emits one
and the same program for these skeletons at every device count: checked here
at 2 layers for m = 1 (planned now), 2 and 4 (reference goldens), and for the
12-layer bench plans at m = 2, 4, 8 (reference goldens).  The bench's plan
files themselves are the reference planner's output (tests/golden/
make_golden.py); their shard tables and ratios are re-derived here from the
program with the LP and the rounding rule, which is fast, while the full
12-layer re-plan (60-170 s each) runs with HAP_SLOW_TESTS=1
(tests/test_planner.py)."""
import json
import os

import pytest

import goldens
from paper_2401_05965_b200 import ClusterSpec, alternate, workloads
from paper_2401_05965_b200.cli import plan_document


def _core(instrs):
    return [{k: v for k, v in i.items() if k not in ("flops", "elements", "sharded")} for i in instrs]


@pytest.mark.parametrize("gname", ["bert2_b2", "moe2_b2"])
def test_planner_emits_the_same_program_at_every_device_count(gname):
    g = goldens.graph(gname)
    spec = ClusterSpec.from_dict(workloads.cluster_doc([148]))
    m1 = plan_document(g, spec, alternate(g, spec))
    for cname in ("b200x2", "b200x4"):
        assert _core(m1["program"]["instrs"]) == _core(goldens.plan(gname, cname)["program"]["instrs"])


@pytest.mark.parametrize("stem", ["bert12", "moe12"])
def test_bench_plans_share_one_program(stem):
    per_gpu = {"bert12": 64, "moe12": 2}[stem]
    docs = [goldens.plan(f"{stem}_b{per_gpu * n}", f"b200x{n}") for n in (2, 4, 8)]
    for d in docs[1:]:
        assert _core(d["program"]["instrs"]) == _core(docs[0]["program"]["instrs"])


@pytest.mark.parametrize("stem", ["bert12", "moe12"])
def test_n1_bench_program_is_the_planned_program(stem):
    per_gpu = {"bert12": 64, "moe12": 2}[stem]
    g = workloads.bert(layers=12, batch=per_gpu) if stem == "bert12" else workloads.moe_stack(layers=12, batch=per_gpu)
    doc = goldens.plan(f"{stem}_b{per_gpu * 2}", "b200x2")
    prog, table, ratios = workloads.planned_program(g, 1, doc)
    assert [i.to_json() for i in prog.instrs] and ratios == (1.0,)
    assert _core([i.to_json() for i in prog.instrs]) == _core(doc["program"]["instrs"])
    assert table[("x0", 0)] == [per_gpu * 128]
    assert all(sizes == [g.producer(ref).shape[axis]] for (ref, axis), sizes in table.items())


@pytest.mark.parametrize("name", ["bert12_b128.b200x2", "bert12_b256.b200x4", "bert12_b512.b200x8",
                                  "moe12_b4.b200x2", "moe12_b8.b200x4", "moe12_b16.b200x8"])
def test_bench_plan_ratios_and_shards_rederive(name):
    """The bench plans' ratios, shard tables and cost estimate follow from
    their program by the planner's own alternating loop (optimizer_loop),
    with the A* synthesis step replaced by the golden program: the LP
    (load_balancer), the rounding (sharding) and the cost model reproduce
    the reference's document byte for byte except the search statistics."""
    from paper_2401_05965_b200.program import DistributedProgram
    from paper_2401_05965_b200.synthesizer import SynthesisResult

    gname, cname = name.rsplit(".", 1)
    g = goldens.graph(gname)
    spec = ClusterSpec.from_dict(goldens.load_json("clusters", f"{cname}.json"))
    doc = goldens.plan(gname, cname)
    prog = DistributedProgram.from_json(doc["program"])

    def synth(*_args):
        return SynthesisResult(program=prog, cost_s=0.0, complete=True, optimal=True, exhausted=False,
                               expansions=0, generated=0, purged=0)

    mine = plan_document(g, spec, alternate(g, spec, synth_fn=synth))
    for key in doc:
        if key != "loop":
            assert json.dumps(mine[key], sort_keys=True) == json.dumps(doc[key], sort_keys=True), key
