"""Generate the golden fixtures by running the *reference* package.

Run in the build container only (it imports the read-only reference from
/root/reference/pkg); the outputs are committed so that tests, smoke() and
bench.py never need the reference at run time.

    python tests/golden/make_golden.py            # corpus + parity plans
    python tests/golden/make_golden.py --bench    # also the 12-layer bench plans (slow)

Writes, under tests/golden/:
  graphs/<name>.json              graph documents (reference corpus + workloads)
  clusters/<name>.json            cluster specs
  plans/<graph>.<cluster>.json    reference plan documents (cli.plan_document)
  values/<graph>.<cluster>.npz    seeded inputs, reference per-device losses,
                                  single-device loss, and every distributed
                                  tensor the reference interpreter realises
                                  (seed 0), named env:<did>:<device>
  grads/<graph>.npz               central-difference gradients of the
                                  reference run_single w.r.t. every source
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
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
sys.path.insert(0, REPO)

import corpus as ref_corpus  # noqa: E402  (reference test corpus)
from shardplan import (ClusterSpec, alternate, build_shard_table,  # noqa: E402
                       graph_from_dict)
from shardplan.cli import plan_document  # noqa: E402
from shardplan.interpreter import (execute_instruction, materialize_loss,  # noqa: E402
                                   random_inputs, run_single)
from shardplan.synthesizer import DistributedProgram  # noqa: E402
from shardplan.cost_model import ShardingRatios, SegmentAssignment  # noqa: E402

from paper_2401_05965_b200 import workloads  # noqa: E402

SEEDS = (0, 1, 2)


def _dump(path: str, obj) -> None:
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(json.dumps(obj, indent=2) + "\n")


def reference_env(program, m, inputs, table):
    """Run the reference interpreter instruction by instruction, keeping env."""
    env: dict = {}
    for instr in program.instrs:
        execute_instruction(instr, env, m, inputs, table)
    return env, materialize_loss(env, program.loss, m)


SMALL = 1 << 16   # element budget for storing arrays verbatim


def _sha(value) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(value, dtype=np.float64).tobytes()).hexdigest()


def plan_case(gname: str, gdoc: dict, cname: str, cdoc: dict, values: bool = True,
              scaled: bool = False, seeds=SEEDS) -> None:
    g = graph_from_dict(gdoc)
    spec = ClusterSpec.from_dict(cdoc)
    t0 = time.time()
    res = alternate(g, spec)
    doc = plan_document(g, spec, res)
    _dump(os.path.join(HERE, "plans", f"{gname}.{cname}.json"), doc)
    print(f"plan {gname}.{cname}: cost {doc['estimate']['total_s']} "
          f"ratios {doc['ratios']} ({time.time() - t0:.1f}s)", flush=True)
    if not values:
        return
    # Execute exactly what the plan file says (canonical ratios + table).
    ratios = ShardingRatios(rows=tuple(tuple(r) for r in doc["ratios"]))
    assignment = SegmentAssignment(segment_of=dict(doc["segment_of"]), count=doc["segments"])
    table = build_shard_table(g, ratios, assignment)
    program = DistributedProgram.from_json(doc["program"])
    arrays = {"scaled": np.array(scaled)}
    for seed in seeds:
        if scaled:
            inputs = workloads.synthetic_inputs(g, seed, scaled=True)
        else:
            inputs = random_inputs(g, np.random.default_rng(seed))
        env, losses = reference_env(program, spec.m, inputs, table)
        small = sum(v.size for v in inputs.values()) <= SMALL
        for name, value in inputs.items():
            if small:
                arrays[f"seed{seed}:input:{name}"] = value
            arrays[f"seed{seed}:sha:{name}"] = np.array(_sha(value))
        arrays[f"seed{seed}:losses"] = np.array([float(v) for v in losses])
        arrays[f"seed{seed}:single"] = np.array(float(run_single(g, inputs)))
        if seed == seeds[0]:
            total = sum(v.size for insts in env.values() for v in insts)
            if total <= SMALL:
                for did, insts in env.items():
                    for dev, value in enumerate(insts):
                        arrays[f"env:{did}:{dev}"] = np.asarray(value)
    path = os.path.join(HERE, "values", f"{gname}.{cname}.npz")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez_compressed(path, **arrays)


def enumerated_cases(per_case: int = 10) -> None:
    """Programs WITH collectives: the planner's corpus plans are all
    communication-free, so every complete program the reference enumerates
    (synthesizer.enumerate_all_complete) is grouped by its collective
    signature and the first of each group (canonical order) kept, with the
    reference interpreter's outputs on seeded inputs."""
    from shardplan import build_theory, single_segment
    from shardplan.synthesizer import enumerate_all_complete

    names = ["matmul_reduce", "two_reduce_rows", "two_reduce_cols", "binary_add",
             "matmul_unary", "identity_after_reduce", "self_add", "rank1_mul"]
    if args.moe:
        moe_plans(bench=args.bench)
        return
    clusters = {"homog2": ref_corpus.HOMOG2, "hetero2": ref_corpus.HETERO2,
                "skew2": ref_corpus.SKEW2, "homog3": ref_corpus.HOMOG3}
    for gname in names:
        gdoc = ref_corpus.CORPUS[gname]
        g = graph_from_dict(gdoc)
        for cname, cdoc in clusters.items():
            spec = ClusterSpec.from_dict(cdoc)
            B = ShardingRatios.proportional_to_flops(spec)
            th = build_theory(g, spec.m, guards=True, fuse=False)
            progs = enumerate_all_complete(g, th, spec, B, max_len=7 if spec.m == 2 else 6)
            groups: dict = {}
            for instrs in progs:
                sig = tuple((i.kind, i.axis, i.axis2) for i in instrs if i.is_comm)
                if not sig:
                    continue
                canon = ";".join(i.canonical() for i in instrs)
                if sig not in groups or canon < groups[sig][0]:
                    groups[sig] = (canon, instrs)
            chosen = [groups[s][1] for s in sorted(groups, key=lambda s: (len(s), str(s)))][:per_case]
            table = build_shard_table(g, B, single_segment(g))
            for idx, instrs in enumerate(chosen):
                program = DistributedProgram(instrs=instrs, loss=g.loss)
                doc = {"devices": spec.m, "ratios": [list(r) for r in B.rows],
                       "shard_table": {f"{r}:{a}": sizes for (r, a), sizes in sorted(table.items())},
                       "program": program.to_json()}
                stem = f"{gname}.{cname}.p{idx}"
                _dump(os.path.join(HERE, "programs", f"{stem}.json"), doc)
                arrays = {}
                for seed in (0, 1):
                    inputs = random_inputs(g, np.random.default_rng(seed))
                    env, losses = reference_env(program, spec.m, inputs, table)
                    for name, value in inputs.items():
                        arrays[f"seed{seed}:input:{name}"] = value
                    arrays[f"seed{seed}:losses"] = np.array([float(v) for v in losses])
                    if seed == 0:
                        for did, insts in env.items():
                            for dev, value in enumerate(insts):
                                arrays[f"env:{did}:{dev}"] = np.asarray(value)
                np.savez_compressed(os.path.join(HERE, "programs", f"{stem}.npz"), **arrays)
            print(f"programs {gname}.{cname}: {len(chosen)} of {len(groups)} signatures", flush=True)


def planner_goldens() -> None:
    """Reference planner internals on the corpus: theory digests, search
    statistics under every optimisation toggle, LP solutions, rounding,
    segmentation and exhaustive-enumeration minima (planner restatement pins)."""
    import hashlib
    import itertools

    from shardplan import (ShardingRatios, assign_segments, build_theory, enumerate_programs,
                           optimize_ratios, round_shards, single_segment, synthesize)
    from shardplan.load_balancer import SegmentProblem, build_lp, lp_solve
    from shardplan.synthesizer import SearchConfig
    from shardplan.theory import theory_to_json

    out: dict = {"theory": {}, "search": {}, "enumerate": {}, "lp": [], "round": [], "segments": {},
                 "ratios": {}}
    homog2 = ClusterSpec.from_dict(ref_corpus.HOMOG2)
    for name, doc in ref_corpus.CORPUS.items():
        g = graph_from_dict(doc)
        for guards, fuse in itertools.product((False, True), repeat=2):
            js = json.dumps(theory_to_json(build_theory(g, 2, guards=guards, fuse=fuse)), sort_keys=True)
            out["theory"][f"{name}:{int(guards)}{int(fuse)}"] = hashlib.sha256(js.encode()).hexdigest()
        B = ShardingRatios.uniform(2)
        for guards, fuse, prune in itertools.product((False, True), repeat=3):
            th = build_theory(g, 2, guards=guards, fuse=fuse)
            res = synthesize(g, th, homog2, B, cfg=SearchConfig(prune_properties=prune))
            out["search"][f"{name}:{int(guards)}{int(fuse)}{int(prune)}"] = {
                "cost": res.cost_s, "expansions": res.expansions, "generated": res.generated,
                "purged": res.purged, "program": res.program.canonical()}
        en = enumerate_programs(g, build_theory(g, 2, guards=False, fuse=False), homog2, B)
        out["enumerate"][name] = {"cost": en.cost_s, "explored": en.explored,
                                  "complete": en.complete_states, "program": en.program.canonical()}
        for k in range(1, min(4, len(g.nodes)) + 1):
            out["segments"][f"{name}:{k}"] = assign_segments(g, k).segment_of
        for cname in ("hetero2", "skew2", "homog3"):
            spec = ClusterSpec.from_dict(getattr(ref_corpus, cname.upper()))
            res = synthesize(g, build_theory(g, spec.m), spec, ShardingRatios.proportional_to_flops(spec))
            out["ratios"][f"{name}:{cname}"] = [list(r) for r in optimize_ratios(res.program, g, spec).rows]
    rng = np.random.default_rng(5)
    for i in range(40):
        m = 2 + i % 3
        stages = int(rng.integers(1, 4))
        prob = SegmentProblem(row_index=0, m=m, comp_a=[rng.uniform(0.0, 4.0, m) for _ in range(stages)],
                              comp_c=[rng.uniform(0.0, 1.0, m) for _ in range(stages)],
                              slope_M=float(rng.uniform(0.0, 3.0)) if i % 3 else 0.0,
                              linear_B=rng.uniform(0.0, 2.0, m), const_s=float(rng.uniform(0.0, 1.0)))
        sol = lp_solve(build_lp(prob))
        out["lp"].append({"m": m, "comp_a": [a.tolist() for a in prob.comp_a],
                          "comp_c": [c.tolist() for c in prob.comp_c], "slope_M": prob.slope_M,
                          "linear_B": prob.linear_B.tolist(), "const_s": prob.const_s,
                          "status": sol.status, "x": sol.x.tolist(), "objective": sol.objective})
    for i in range(200):
        m = 1 + i % 5
        row = tuple(float(v) for v in rng.dirichlet(np.ones(m)))
        extent = int(rng.integers(0, 40))
        out["round"].append({"extent": extent, "row": list(row), "sizes": round_shards(extent, row)})
    _dump(os.path.join(HERE, "planner.json"), out)
    print("planner goldens written", flush=True)


def fd_gradients(gname: str, gdoc: dict, eps: float = 1e-5) -> None:
    g = graph_from_dict(gdoc)
    inputs = random_inputs(g, np.random.default_rng(0))
    out = {}
    for name, value in inputs.items():
        grad = np.zeros_like(value)
        flat = value.reshape(-1)
        gflat = grad.reshape(-1)
        for i in range(flat.size):
            keep = flat[i]
            flat[i] = keep + eps
            up = float(run_single(g, inputs))
            flat[i] = keep - eps
            down = float(run_single(g, inputs))
            flat[i] = keep
            gflat[i] = (up - down) / (2 * eps)
        out[f"grad:{name}"] = grad
        out[f"input:{name}"] = value.copy()
    path = os.path.join(HERE, "grads", f"{gname}.npz")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez_compressed(path, **out)


def moe_plans(bench: bool) -> None:
    """configs[4]: BERT-MoE stack (2 SiLU experts per layer, residual merge),
    2 sequences of 128 tokens per GPU — the regime where the cost model picks
    sufficient-factor broadcasting at 2 and 4 GPUs and all-reduce at 8."""
    for n in (2, 4):
        cdoc = workloads.cluster_doc(workloads.sm_caps(n), fitted=False)
        gdoc = workloads.moe_stack_doc(layers=2, batch=2, seq=64)
        _dump(os.path.join(HERE, "graphs", "moe2_b2.json"), gdoc)
        plan_case("moe2_b2", gdoc, f"b200x{n}", cdoc, scaled=True, seeds=(0,))
    if bench:
        for n in (2, 4, 8):
            cdoc = workloads.cluster_doc(workloads.sm_caps(n), fitted=False)
            gdoc = workloads.moe_stack_doc(layers=12, batch=2 * n, seq=128)
            plan_case(f"moe12_b{2 * n}", gdoc, f"b200x{n}", cdoc, values=False)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", action="store_true", help="also plan the 12-layer bench graphs")
    ap.add_argument("--moe", action="store_true", help="only the MoE-stack plans (configs[4])")
    args = ap.parse_args()

    if args.moe:
        moe_plans(bench=args.bench)
        return
    clusters = {"homog2": ref_corpus.HOMOG2, "homog3": ref_corpus.HOMOG3,
                "hetero2": ref_corpus.HETERO2, "skew2": ref_corpus.SKEW2}
    for cname, cdoc in clusters.items():
        _dump(os.path.join(HERE, "clusters", f"{cname}.json"), cdoc)
    graphs = dict(ref_corpus.CORPUS)
    graphs["chain4"] = ref_corpus.chain_graph(4)
    for gname, gdoc in graphs.items():
        _dump(os.path.join(HERE, "graphs", f"{gname}.json"), gdoc)
        for cname, cdoc in clusters.items():
            plan_case(gname, gdoc, cname, cdoc)
        fd_gradients(gname, gdoc)

    enumerated_cases()
    planner_goldens()

    # configs[0]: 2-layer MLP, hidden 1024, batch 64, two devices at speed 1:2.
    mlp_cluster = workloads.cluster_doc([148, 296], bytes_per_element=2, fitted=False)
    mlp_cluster["devices"] = [{"flops": 1e14}, {"flops": 2e14}]
    _dump(os.path.join(HERE, "clusters", "ratio12.json"), mlp_cluster)
    _dump(os.path.join(HERE, "graphs", "mlp.json"), workloads.mlp_doc())
    plan_case("mlp", workloads.mlp_doc(), "ratio12", mlp_cluster, scaled=True)

    # Small BERT skeletons on SM-capped B200 clusters (parity-test scale).
    for n in (2, 4):
        cdoc = workloads.cluster_doc(workloads.sm_caps(n), fitted=False)
        _dump(os.path.join(HERE, "clusters", f"b200x{n}.json"), cdoc)
        gdoc = workloads.bert_doc(layers=2, batch=2, seq=128)
        _dump(os.path.join(HERE, "graphs", "bert2_b2.json"), gdoc)
        plan_case("bert2_b2", gdoc, f"b200x{n}", cdoc, scaled=True, seeds=(0,))

    if args.bench:
        # Bench workload: BERT-base skeleton, 64 sequences of 128 tokens per GPU.
        # N=1 is planned by the package planner: the reference search at m=1
        # ties on every sharding choice and its O(expansions^2) dominance scan
        # does not finish at 12 layers ("planning at m=1").
        for n in (2, 4, 8):
            cdoc = workloads.cluster_doc(workloads.sm_caps(n), fitted=False)
            _dump(os.path.join(HERE, "clusters", f"b200x{n}.json"), cdoc)
            gdoc = workloads.bert_doc(layers=12, batch=64 * n, seq=128)
            plan_case(f"bert12_b{64 * n}", gdoc, f"b200x{n}", cdoc, values=False)


if __name__ == "__main__":
    main()
