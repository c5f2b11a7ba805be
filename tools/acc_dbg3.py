import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import test_gpu_kernels as T
for i in range(3):
    try:
        T.test_matmul_batch_grouped_and_summed(0, 0, torch.bfloat16); print("pass", i)
    except AssertionError as e:
        print("FAIL", i, str(e)[:80])
