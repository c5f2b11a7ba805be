"""Per-launch GEMM table of the bench step (N=1): every tcgen05 GEMM launch
the executor compiled for the workload, each captured alone R times in one
CUDA graph and replayed (GPU time per launch, no host cost), next to cuBLAS
(torch.matmul, bf16 out, same orientation and shapes, captured the same way).

    python tools/gemm_step_table.py [--workload bert|moe|vitmoe] [--json PATH]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2401_05965_b200 import _lib, workloads  # noqa: E402
from paper_2401_05965_b200.executor import ExecConfig, Executor, LocalGroup  # noqa: E402

R = 20


def graph_us(fn, stream, reps=R, iters=5):
    with torch.cuda.stream(stream):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(reps):
            fn()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            g.replay()
            e0.record(stream)
            for _ in range(iters):
                g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / (iters * reps))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bert")
    ap.add_argument("--json")
    ap.add_argument("--no-cublas", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    wl = bench.WORKLOADS[args.workload]
    g = bench._graph(args.workload, wl["per_gpu_batch"])
    doc = bench._plan_doc(args.workload, 1)
    prog, table, ratios = workloads.planned_program(g, 1, doc)
    ex = Executor(prog, 1, table, {n.id: n.shape for n in g.sources()}, group=LocalGroup(1),
                  config=ExecConfig(dtype="bf16", sm_caps=[148], lr=bench.LR), device=dev)
    ex.load(workloads.synthetic_inputs(g, 0, scaled=True))
    ex.step()
    torch.cuda.synchronize()
    s = ex.stream
    rows = []
    for phase, ops in (("fwd", ex.ops_fwd), ("bwd", ex.ops_bwd)):
        for op in ops:
            if op.gemm is None:
                continue
            members = op.gemm.get("members", [op.gemm])
            run = (lambda op=op: _lib.check(op.fn(*op.args[:-1], s.cuda_stream), op.what))
            us = graph_us(run, s)
            flops = sum(2 * m["M"] * m["N"] * m["K"] for m in members)
            cub = None
            if not args.no_cublas:
                mats = []
                for m in members:
                    a = torch.randn(m["M"], m["K"], device=dev, dtype=torch.bfloat16)
                    b = torch.randn(m["K"], m["N"], device=dev, dtype=torch.bfloat16)
                    if m.get("transA"):
                        a = torch.randn(m["K"], m["M"], device=dev, dtype=torch.bfloat16).t()
                    if not m.get("transB", 0) == 0:
                        b = torch.randn(m["N"], m["K"], device=dev, dtype=torch.bfloat16).t()
                    mats.append((a, b))
                cub = graph_us(lambda: [torch.matmul(a, b) for a, b in mats], s)
            key = op.gemm
            rows.append({"phase": phase, "what": op.what, "members": len(members),
                         "M": key["M"], "N": key["N"], "K": key["K"],
                         "transA": key.get("transA", 0), "transB": key.get("transB", 0),
                         "epi": key.get("epi", 0), "out": "bf16" if key["out_dt"] else "f32",
                         "us": round(us, 2), "tflops": round(flops / us / 1e6, 1),
                         "cublas_us": None if cub is None else round(cub, 2)})
            print(json.dumps(rows[-1]), flush=True)
    tot = sum(r["us"] for r in rows)
    cub = sum(r["cublas_us"] or 0 for r in rows)
    flops = sum(r["tflops"] * r["us"] * 1e6 for r in rows)
    print(f"launches {len(rows)}  ours {tot:.1f} us  cuBLAS {cub:.1f} us  ours {flops / tot / 1e6:.0f} TF/s")
    if args.json:
        with open(args.json, "w") as fh:
            json.dump({"workload": args.workload, "rows": rows, "ours_us": tot, "cublas_us": cub}, fh, indent=1)


if __name__ == "__main__":
    main()
