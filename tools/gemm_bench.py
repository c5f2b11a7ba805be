"""Per-shape GEMM throughput of hap_matmul vs cuBLAS (torch.matmul) on the
GEMMs of one BERT-skeleton train step (T = 8192 tokens)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2401_05965_b200 import _lib
from paper_2401_05965_b200._lib import BF16, F32, check
L = _lib.lib(); dev = torch.device("cuda")
T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
shapes = [  # (name, M, N, K, ta, tb, out)
    ("fwd qkvo", T, 768, 768, 0, 0, torch.bfloat16),
    ("fwd f1", T, 3072, 768, 0, 0, torch.bfloat16),
    ("fwd f2", T, 768, 3072, 0, 0, torch.bfloat16),
    ("dA qkvo", T, 768, 768, 0, 1, torch.bfloat16),
    ("dA f1", T, 768, 3072, 0, 1, torch.bfloat16),
    ("dA f2", T, 3072, 768, 0, 1, torch.bfloat16),
    ("dW qkvo", 768, 768, T, 1, 0, torch.float32),
    ("dW f1", 768, 3072, T, 1, 0, torch.float32),
    ("dW f2", 3072, 768, T, 1, 0, torch.float32),
    ("square 8k", 8192, 8192, 8192, 0, 0, torch.bfloat16),
]
s = torch.cuda.Stream()
for name, M, N, K, ta, tb, out in shapes:
    a = torch.randn((K, M) if ta else (M, K), device=dev).to(torch.bfloat16)
    b = torch.randn((N, K) if tb else (K, N), device=dev).to(torch.bfloat16)
    c = torch.empty((M, N), device=dev, dtype=out)
    args = (a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb, c.data_ptr(), N, M, N, K, BF16,
            BF16 if out == torch.bfloat16 else F32, 0, 0, s.cuda_stream)
    reps = 50 if M * N * K < 1e11 else 10
    for _ in range(3): check(L.hap_matmul(*args))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps): L.hap_matmul(*args)
    e1.record(s); torch.cuda.synchronize()
    ours = e0.elapsed_time(e1) / reps
    A = a.t() if ta else a; B = b.t() if tb else b
    with torch.cuda.stream(s):
        for _ in range(3): torch.matmul(A, B)
        e0.record(s)
        for _ in range(reps): torch.matmul(A, B)
        e1.record(s)
    torch.cuda.synchronize()
    cub = e0.elapsed_time(e1) / reps
    fl = 2 * M * N * K
    print(f"{name:10s} M={M:5d} N={N:5d} K={K:5d} ta={ta} tb={tb}  ours {ours*1e3:8.1f} us {fl/ours/1e9:7.1f} TF/s | cublas {cub*1e3:8.1f} us {fl/cub/1e9:7.1f} TF/s")
