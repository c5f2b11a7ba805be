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

# HAP_PROFILE_WORKLOAD=moe profiles the BERT-MoE stack (2 sequences) instead.
if os.environ.get("HAP_PROFILE_WORKLOAD") == "moe":
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
        key = (f"{op.what} x{len(ms)}{' sum' if op.gemm.get('sum_k') else ''} M={ms[0]['M']} N={ms[0]['N']} "
               f"K={ms[0]['K']} tA={ms[0]['transA']} tB={ms[0]['transB']} out={'bf16' if ms[0]['out_dt'] else 'f32'}")
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
