"""configs[3] (ViT-MoE, expert-sharded FFN, uneven all-gather / reduce-scatter)
fixtures, made by running the *reference* package.

The reference planner never emits an expert-sharded program for these
graphs: its forward-only sum loss prices data parallelism as free of
communication.  The program is instead taken from the reference's own
program space:

1. space.json — the reference's enumerate_all_complete (synthesizer.py:538)
   over one expert-FFN block (x0 -> relu -> W1 / SiLU / W2 -> residual ->
   loss) on 2 devices finds the expert-sliced pattern the executor runs in
   every ViT-MoE layer: all-gather the block input along tokens, W1
   column-sharded, W2 row-sharded, partial sums, reduce-scatter back to
   token rows.
2. plans/vitmoe*.json — workloads.expert_sharded_program (that pattern in
   every layer, attention data parallel) with ratios, shard table and
   estimate from the reference's alternate() whose synthesis step is fixed
   to the program (so the LP, rounding and cost model are the reference's);
   plan_document from the reference.
3. values/vitmoe2_*.npz — the reference interpreter's losses and every
   realised tensor on seeded inputs for the small parity graph, and the
   reference check_equivalence at rtol 1e-9.

    python tests/golden/make_vit_moe.py [--bench]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

from shardplan import ClusterSpec, alternate, build_shard_table, build_theory, graph_from_dict  # noqa: E402
from shardplan.cli import plan_document  # noqa: E402
from shardplan.cost_model import SegmentAssignment, ShardingRatios  # noqa: E402
from shardplan.interpreter import check_equivalence, run_single  # noqa: E402
from shardplan.synthesizer import DistributedProgram, SynthesisResult, enumerate_all_complete  # noqa: E402

from make_golden import _dump, _sha, reference_env  # noqa: E402
from paper_2401_05965_b200 import workloads  # noqa: E402

SMALL = dict(layers=2, experts=2, images=2, tokens=32, hidden=64, ffn=256)
BENCH_IMAGES_PER_GPU = 16


def program_space() -> None:
    n = workloads._n
    nodes = [n("x0", "Placeholder", [16, 8]), n("x", "ElemwiseUnary", [16, 8], ["x0"], tag="relu"),
             n("W1", "Parameter", [8, 32]), n("f1", "MatMul", [16, 32], ["x", "W1"]),
             n("s1", "ElemwiseUnary", [16, 32], ["f1"], tag="sigmoid"),
             n("g", "ElemwiseBinary", [16, 32], ["f1", "s1"], tag="mul"),
             n("W2", "Parameter", [32, 8]), n("y", "MatMul", [16, 8], ["g", "W2"]),
             n("x2", "ElemwiseBinary", [16, 8], ["x", "y"], tag="add"), n("loss", "Reduce", [], ["x2"], dims="all")]
    gdoc = {"nodes": nodes, "loss": "loss"}
    g = graph_from_dict(gdoc)
    spec = ClusterSpec.from_dict(workloads.cluster_doc([148, 104], fitted=False))
    B = ShardingRatios.proportional_to_flops(spec)
    t0 = time.time()
    progs = enumerate_all_complete(g, build_theory(g, 2), spec, B, max_len=13)
    target = ["x0@shard0<-placeholder_shard/x0/d=0()", "x@shard0<-elemwise_unary/x(x0@shard0)",
              "x@full<-all_gather/x/d=0(x@shard0)", "W1@shard1<-parameter_shard/W1/d=1()",
              "f1@shard1<-matmul/f1(x@full,W1@shard1)", "s1@shard1<-elemwise_unary/s1(f1@shard1)",
              "g@shard1<-elemwise_binary/g(f1@shard1,s1@shard1)", "W2@shard0<-parameter_shard/W2/d=0()",
              "y@partial<-matmul/y(g@shard1,W2@shard0)", "y@shard0<-reduce_scatter/y/d=0(y@partial)",
              "x2@shard0<-elemwise_binary/x2(x@shard0,y@shard0)", "loss@partial<-reduce/loss(x2@shard0)"]
    hits = [[i.canonical() for i in p] for p in progs if {i.canonical() for i in p} == set(target)]
    assert hits, "the expert-sliced FFN program is not in the reference program space"
    doc = {"graph": gdoc, "cluster": "b200x2 (caps 148/104)", "max_len": 13, "programs_enumerated": len(progs),
           "expert_sliced_program": sorted(hits)[0], "seconds": round(time.time() - t0, 1)}
    _dump(os.path.join(HERE, "vit_moe", "space.json"), doc)
    print(f"program space: {len(progs)} complete programs, expert-sliced pattern found ({len(hits)} orders)")


def plan(gname: str, gdoc: dict, cname: str, cdoc: dict) -> dict:
    g = graph_from_dict(gdoc)
    spec = ClusterSpec.from_dict(cdoc)
    mine = workloads.expert_sharded_program(workloads.graph_from_dict(gdoc))
    prog = DistributedProgram.from_json(mine.to_json())
    # every instruction is one of the REFERENCE theory's Hoare triples and its
    # precondition holds where it runs (theory.py, guards on, sources unfused)
    from shardplan.theory import build_theory as ref_theory, merge_post

    th = ref_theory(g, spec.m, fuse=False)
    index: dict = {}
    for t in th.triples:
        if len(t.instrs) == 1:
            index.setdefault(t.instrs[0].canonical(), []).append(t)
    props = frozenset(th.initial_props)
    for ins in prog.instrs:
        ts = [t for t in index.get(ins.canonical(), []) if t.pre <= props and t.instrs[0] == ins]
        assert ts, f"{ins.canonical()} is not a reference-theory step here"
        props = merge_post(props, ts[0].post)

    def synth(*_args):
        return SynthesisResult(program=prog, cost_s=0.0, complete=True, optimal=True, exhausted=False,
                               expansions=0, generated=0, purged=0)

    t0 = time.time()
    doc = plan_document(g, spec, alternate(g, spec, synth_fn=synth))
    _dump(os.path.join(HERE, "plans", f"{gname}.{cname}.json"), doc)
    print(f"plan {gname}.{cname}: ratios {doc['ratios']} estimate {doc['estimate']['total_s']} "
          f"({time.time() - t0:.1f}s)", flush=True)
    return doc


def values(gname: str, gdoc: dict, cname: str, doc: dict) -> None:
    g = graph_from_dict(gdoc)
    ratios = ShardingRatios(rows=tuple(tuple(r) for r in doc["ratios"]))
    assignment = SegmentAssignment(segment_of=dict(doc["segment_of"]), count=doc["segments"])
    table = build_shard_table(g, ratios, assignment)
    program = DistributedProgram.from_json(doc["program"])
    m = int(doc["devices"])
    arrays = {"scaled": np.array(True)}
    inputs = workloads.synthetic_inputs(workloads.graph_from_dict(gdoc), 0, scaled=True)
    env, losses = reference_env(program, m, inputs, table)
    for name, value in inputs.items():
        arrays[f"seed0:input:{name}"] = value
        arrays[f"seed0:sha:{name}"] = np.array(_sha(value))
    arrays["seed0:losses"] = np.array([float(v) for v in losses])
    arrays["seed0:single"] = np.array(float(run_single(g, inputs)))
    for did, insts in env.items():
        for dev, value in enumerate(insts):
            arrays[f"env:{did}:{dev}"] = np.asarray(value)
    rep = check_equivalence(g, program, m, table, trials=3, seed=0, rtol=1e-9)
    assert rep.passed, rep
    path = os.path.join(HERE, "values", f"{gname}.{cname}.npz")
    np.savez_compressed(path, **arrays)
    print(f"values {gname}.{cname}: losses {[float(v) for v in losses]}, reference check_equivalence "
          f"max rel err {rep.max_rel_err:.2e}")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", action="store_true", help="also the 12-layer bench plans")
    ap.add_argument("--no-space", action="store_true")
    args = ap.parse_args()
    if not args.no_space:
        program_space()
    gdoc = workloads.vit_moe_doc(**SMALL)
    _dump(os.path.join(HERE, "graphs", "vitmoe2.json"), gdoc)
    for n in (2, 4):
        cdoc = workloads.cluster_doc(workloads.sm_caps(n), fitted=False)
        doc = plan("vitmoe2", gdoc, f"b200x{n}", cdoc)
        values("vitmoe2", gdoc, f"b200x{n}", doc)
    if args.bench:
        for n in (2, 4, 8):
            cdoc = workloads.cluster_doc(workloads.sm_caps(n), fitted=False)
            plan(f"vitmoe12_b{BENCH_IMAGES_PER_GPU * n}",
                 workloads.vit_moe_doc(layers=12, experts=2, images=BENCH_IMAGES_PER_GPU * n), f"b200x{n}", cdoc)


if __name__ == "__main__":
    main()
