import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import test_gpu_kernels as T
M, N, K = (int(v) for v in sys.argv[1:4])
epi = sys.argv[4]
T.test_gemm_fused_epilogues(M, N, K, 0, 0, epi)
print("ok", M, N, K, epi)
