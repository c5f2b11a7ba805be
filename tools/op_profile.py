"""Per-op GPU time of one training step of the bench workload (N=1), eager
launches bracketed by CUDA events on the executor stream.  Aggregates by op
(and GEMM shape) and compares the sum with the CUDA-graph step time."""
import collections
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2401_05965_b200 import api, workloads  # noqa: E402
from paper_2401_05965_b200.executor import ExecConfig, Executor, LocalGroup  # noqa: E402

# HAP_PROFILE_WORKLOAD=moe profiles the BERT-MoE stack (2 sequences) instead;
# HAP_PROFILE_WORKLOAD=vitmoe2 the ViT-MoE 2-GPU expert-sharded plan with both
# ranks on this GPU (LocalGroup, SM caps 148 / 104): per-op costs of the
# multi-GPU program without the peers.
wl = os.environ.get("HAP_PROFILE_WORKLOAD")
if wl == "vitmoe2":
    import bench
    from paper_2401_05965_b200.program import DistributedProgram
    from paper_2401_05965_b200.sharding import table_from_plan

    g = bench._graph("vitmoe", bench.WORKLOADS["vitmoe"]["per_gpu_batch"] * 2)
    doc = bench._plan_doc("vitmoe", 2)
    ex = Executor(DistributedProgram.from_json(doc["program"]), 2, table_from_plan(doc),
                  {n.id: n.shape for n in g.sources()}, group=LocalGroup(2),
                  config=ExecConfig(dtype="bf16", lr=1e-11, sm_caps=[148, 104]))
else:
    if wl == "moe":
        g = workloads.moe_stack(layers=12, batch=2, seq=128)
    else:
        g = workloads.bert(layers=12, batch=64, seq=128)
    ex = Executor(api.single_device_program(g), 1, {}, {n.id: n.shape for n in g.sources()}, group=LocalGroup(1),
                  config=ExecConfig(dtype="bf16", lr=1e-11))
ex.load(workloads.synthetic_inputs(g, 0, scaled=True))
ops = ex.ops_fwd + ex.ops_bwd + ex.ops_upd
for _ in range(3):
    ex.step()
torch.cuda.synchronize()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(ops) + 1)]
with torch.cuda.stream(ex.stream):
    evs[0].record(ex.stream)
    for op, ev in zip(ops, evs[1:]):
        op.fn(*op.args)
        ev.record(ex.stream)
torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for op, a, b in zip(ops, evs[:-1], evs[1:]):
    key = op.what
    if op.gemm is not None:
        ms = op.gemm.get("members", [op.gemm])
        m0 = ms[0]
        eng = ex.lib.hap_matmul_engine(m0["A"], m0["lda"], m0["transA"], m0["B"], m0["ldb"], m0["transB"], m0["M"],
                                       m0["N"], m0["K"], m0["in_dt"])
        key = (f"{op.what} x{len(ms)}{' sum' if op.gemm.get('sum_k') else ''} M={m0['M']} N={m0['N']} "
               f"K={m0['K']} tA={m0['transA']} tB={m0['transB']} out={'bf16' if m0['out_dt'] else 'f32'} "
               f"epi={m0['epi']} {'simt' if eng else 'tc'}")
    agg[key][0] += 1
    agg[key][1] += a.elapsed_time(b)
total = sum(v[1] for v in agg.values())
ex.capture()
for _ in range(3):
    ex.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(ex.stream)
for _ in range(20):
    ex.step()
e1.record(ex.stream)
torch.cuda.synchronize()
print(f"eager sum of op times {total:.3f} ms over {len(ops)} ops; graph step {e0.elapsed_time(e1) / 20:.3f} ms")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{t:8.3f} ms {t / total:6.1%}  x{n:4d}  {t / n * 1e3:8.1f} us  {k}")
