"""Run one GEMM shape repeatedly (for ncu): python tools/gemm_one.py M N K ta tb [out=bf16|f32] [reps]"""
import sys, torch
sys.path.insert(0, ".")
from paper_2401_05965_b200 import _lib
from paper_2401_05965_b200._lib import BF16, F32, check
M, N, K, ta, tb = (int(v) for v in sys.argv[1:6])
out = torch.float32 if len(sys.argv) > 6 and sys.argv[6] == "f32" else torch.bfloat16
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 5
L = _lib.lib(); dev = torch.device("cuda")
a = torch.randn((K, M) if ta else (M, K), device=dev).to(torch.bfloat16)
b = torch.randn((N, K) if tb else (K, N), device=dev).to(torch.bfloat16)
c = torch.empty((M, N), device=dev, dtype=out)
for _ in range(reps):
    check(L.hap_matmul(a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb, c.data_ptr(), N, M, N, K, BF16,
                       BF16 if out == torch.bfloat16 else F32, 0, 0, 0))
torch.cuda.synchronize()
print("ok")
