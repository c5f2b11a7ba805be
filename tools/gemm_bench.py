"""Per-shape GEMM throughput of the tcgen05 path (heuristic shape choice and
after hap_matmul_tune) vs cuBLAS (torch.matmul) on the GEMM shapes of one
BERT-skeleton train step (T = 8192 tokens).  Prints one line per shape and,
with --json PATH, writes the table."""
import json, sys, torch
sys.path.insert(0, ".")
from paper_2401_05965_b200 import _lib
from paper_2401_05965_b200._lib import BF16, F32, check
L = _lib.lib(); dev = torch.device("cuda")
out_json = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
args_ = [a for a in sys.argv[1:] if not a.startswith("--") and a != out_json]
T = int(args_[0]) if args_ else 8192
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
if "--sweep" in sys.argv:   # fixed cost vs K: intercept = launch + prologue + fill + last epilogue
    shapes = [(f"sweep K={k}", T, n, k, 0, 0, torch.bfloat16) for n in (768, 3072) for k in (64, 128, 256, 768, 1536, 3072)]
s = torch.cuda.Stream()
rows = []


def timeit(fn, reps):
    with torch.cuda.stream(s):
        for _ in range(3): fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps): fn()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, M, N, K, ta, tb, out in shapes:
    a = torch.randn((K, M) if ta else (M, K), device=dev).to(torch.bfloat16)
    b = torch.randn((N, K) if tb else (K, N), device=dev).to(torch.bfloat16)
    c = torch.empty((M, N), device=dev, dtype=out)
    odt = BF16 if out == torch.bfloat16 else F32
    d = _lib.GemmDesc()
    d.A, d.lda, d.transA, d.B, d.ldb, d.transB = a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb
    d.C, d.ldc, d.M, d.N, d.K = c.data_ptr(), N, M, N, K
    arr = (_lib.GemmDesc * 1)(d)
    reps = 50 if M * N * K < 1e11 else 10
    run = lambda: L.hap_matmul_batch(arr, 1, 0, BF16, odt, 0, s.cuda_stream)
    check(run())
    heur = timeit(run, reps)
    check(L.hap_matmul_tune(arr, 1, 0, BF16, odt, 0, s.cuda_stream), "tune")
    tuned = timeit(run, reps)
    A = a.t() if ta else a; B = b.t() if tb else b
    cub = timeit(lambda: torch.matmul(A, B), reps)
    fl = 2 * M * N * K
    tf = lambda ms: fl / ms / 1e9
    rows.append({"name": name, "M": M, "N": N, "K": K, "transA": ta, "transB": tb,
                 "out": "f32" if odt == F32 else "bf16", "heuristic_us": heur * 1e3, "tuned_us": tuned * 1e3,
                 "cublas_us": cub * 1e3, "tuned_tflops": tf(tuned), "cublas_tflops": tf(cub)})
    print(f"{name:10s} M={M:5d} N={N:5d} K={K:5d} ta={ta} tb={tb}  heur {heur*1e3:7.1f} us {tf(heur):7.1f} | "
          f"tuned {tuned*1e3:7.1f} us {tf(tuned):7.1f} TF/s | cublas {cub*1e3:7.1f} us {tf(cub):7.1f} TF/s",
          flush=True)
if out_json:
    with open(out_json, "w") as fh:
        json.dump({"tokens": T, "note": "CUDA events, back-to-back launches on one stream, inputs resident",
                   "rows": rows}, fh, indent=1)
