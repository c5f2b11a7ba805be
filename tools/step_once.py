"""Build the bench executor (N=1) and run a few eager training steps — a
small target for `ncu` (per-kernel counters of one step)."""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2401_05965_b200 import api, workloads  # noqa: E402
from paper_2401_05965_b200.executor import ExecConfig, Executor, LocalGroup  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
if os.environ.get("HAP_PROFILE_WORKLOAD") == "moe":
    g = workloads.moe_stack(layers=12, batch=2, seq=128)
else:
    g = workloads.bert(layers=12, batch=64, seq=128)
ex = Executor(api.single_device_program(g), 1, {}, {n.id: n.shape for n in g.sources()}, group=LocalGroup(1),
              config=ExecConfig(dtype="bf16", lr=1e-11))
ex.load(workloads.synthetic_inputs(g, 0, scaled=True))
gemm_launches = sum(len(op.gemm.get("members", [op.gemm])) > 0 for op in ex.ops_fwd + ex.ops_bwd if op.gemm)
print("gemm launches per step", gemm_launches)
# ncu --profile-from-start off sees only the steps (not the compile-time
# GEMM tuning, which launches thousands of candidate kernels)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(steps):
    ex.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
