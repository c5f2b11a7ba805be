"""Generate the committed GEMM tuning table (paper_2401_05965_b200/tune_b200.txt)
on a B200.

Compiles the executors the bench and smoke() run — BERT (configs[2]) and
BERT-MoE (configs[4]) at the 1/2/4/8-GPU plans, every rank's SM cap, plus the
configs[0] MLP — with autotune="time": every GEMM launch signature is timed
once (hap_matmul_tune: each tile shape / split-K candidate, CUDA-graph timed)
and the fastest kept; the table is then exported.  Multi-GPU plans are
compiled with LocalGroup (all ranks on this GPU): the launch signatures —
shapes, orientation, epilogue, SM cap — are those each rank's process uses.

    python tools/tune_table.py [--out paper_2401_05965_b200/tune_b200.txt] [--gpus 1,2,4,8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    import torch

    from paper_2401_05965_b200 import _lib, workloads
    from paper_2401_05965_b200.cost_model import ClusterSpec
    from paper_2401_05965_b200.executor import ExecConfig, Executor, LocalGroup
    from paper_2401_05965_b200.graph_ir import graph_from_dict
    from paper_2401_05965_b200.program import DistributedProgram
    from paper_2401_05965_b200.sharding import table_from_plan

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=_lib.TUNE_TABLE)
    ap.add_argument("--gpus", default="1,2,4,8")
    ap.add_argument("--workloads", default="bert,moe")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    assert _lib.lib().hap_sm_count() == 148, "the table is for a 148-SM B200"
    _lib.lib().hap_matmul_tune_clear()
    plans = os.path.join(ROOT, "tests", "golden", "plans")
    per_gpu = {"bert": 64, "moe": 2}
    stem = {"bert": "bert12", "moe": "moe12"}
    total = 0
    for wl in args.workloads.split(","):
        for n in [int(x) for x in args.gpus.split(",")]:
            batch = per_gpu[wl] * n
            g = workloads.moe_stack(layers=12, batch=batch, seq=128) if wl == "moe" else \
                workloads.bert(layers=12, batch=batch, seq=128)
            caps = workloads.sm_caps(n)
            shapes = {nd.id: nd.shape for nd in g.sources()}
            k = max(n, 2)
            with open(os.path.join(plans, f"{stem[wl]}_b{per_gpu[wl] * k}.b200x{k}.json")) as fh:
                doc = json.load(fh)
            if n == 1:
                prog, table, ratios = workloads.planned_program(g, 1, doc)
            else:
                prog, table, ratios = (DistributedProgram.from_json(doc["program"]), table_from_plan(doc),
                                       tuple(doc["ratios"][0]))
            cluster = ClusterSpec.from_dict(workloads.cluster_doc(caps))
            ex = Executor(prog, n, table, shapes, group=LocalGroup(n),
                          config=ExecConfig(dtype="bf16", sm_caps=caps, lr=1e-11, cluster=cluster, ratios=ratios,
                                            autotune="time"))
            total += ex.tuned_signatures
            print(f"{wl} N={n}: {ex.tuned_signatures} signatures timed", flush=True)
            ex.close()
            del ex
            torch.cuda.empty_cache()
    with open(os.path.join(ROOT, "tests", "golden", "plans", "mlp.ratio12.json")) as fh:
        doc = json.load(fh)
    with open(os.path.join(ROOT, "tests", "golden", "graphs", "mlp.json")) as fh:
        g = graph_from_dict(json.load(fh))
    ex = Executor(DistributedProgram.from_json(doc["program"]), doc["devices"], table_from_plan(doc),
                  {n.id: n.shape for n in g.sources()}, group=LocalGroup(doc["devices"]),
                  config=ExecConfig(dtype="bf16", sm_caps=[74, 148], autotune="time"))
    total += ex.tuned_signatures
    ex.close()
    text = _lib.export_tune_table()
    with open(args.out, "w") as fh:
        fh.write(text)
    print(f"wrote {args.out}: {text.count(chr(10))} signatures ({total} timed)")


if __name__ == "__main__":
    main()
