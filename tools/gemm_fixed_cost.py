"""GPU-side fixed cost of one tcgen05 GEMM launch, measured inside a CUDA
graph (no host launch cost): R launches of the same GEMM captured in one
graph, replayed, CUDA events around the replay.  Compared with an empty
kernel (hap_fill of one element) in the same setup.  Shapes: the smallest
unit (one 256-row tile), the BERT N=768 and N=3072 forward shapes over a K
sweep, and the MoE (256-token) shapes.  Prints a table; --json PATH writes it."""
import json, sys, torch
sys.path.insert(0, ".")
from paper_2401_05965_b200 import _lib
from paper_2401_05965_b200._lib import BF16, F32, check

L = _lib.lib(); dev = torch.device("cuda")
out_json = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
s = torch.cuda.Stream()
R = 20


def graph_time(fn, reps=R, iters=10):
    with torch.cuda.stream(s):
        for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(iters): g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (iters * reps)   # us per launch


rows = []
one = torch.zeros(16, device=dev)
empty_us = graph_time(lambda: check(L.hap_fill(one.data_ptr(), F32, 1.0, 1, s.cuda_stream)))
print(f"empty kernel (hap_fill n=1): {empty_us:.2f} us per launch in a graph", flush=True)
rows.append({"name": "empty", "us": empty_us})

shapes = [("one tile", 256, 192, 64, 0, 0), ("one tile K=768", 256, 192, 768, 0, 0)]
shapes += [(f"bert N=768 K={k}", 8192, 768, k, 0, 0) for k in (64, 768, 3072)]
shapes += [(f"bert N=3072 K={k}", 8192, 3072, k, 0, 0) for k in (64, 768)]
shapes += [("moe f1", 256, 3072, 768, 0, 0), ("moe y", 256, 768, 3072, 0, 0),
           ("moe dW1", 768, 3072, 256, 1, 0), ("moe dx", 256, 768, 3072, 0, 1)]
for name, M, N, K, ta, tb in shapes:
    a = torch.randn((K, M) if ta else (M, K), device=dev).to(torch.bfloat16)
    b = torch.randn((N, K) if tb else (K, N), device=dev).to(torch.bfloat16)
    out = torch.float32 if ta else torch.bfloat16
    c = torch.empty((M, N), device=dev, dtype=out)
    odt = F32 if ta else BF16
    d = _lib.GemmDesc()
    d.A, d.lda, d.transA, d.B, d.ldb, d.transB = a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb
    d.C, d.ldc, d.M, d.N, d.K = c.data_ptr(), N, M, N, K
    arr = (_lib.GemmDesc * 1)(d)
    run = lambda: check(L.hap_matmul_batch(arr, 1, 0, BF16, odt, 0, s.cuda_stream))
    run()
    heur = graph_time(run)
    check(L.hap_matmul_tune(arr, 1, 0, BF16, odt, 0, s.cuda_stream), "tune")
    tuned = graph_time(run)
    A = a.t() if ta else a; B = b.t() if tb else b
    cub = graph_time(lambda: torch.matmul(A, B))
    fl = 2 * M * N * K
    byts = 2 * (M * K + K * N) + (4 if ta else 2) * M * N
    rows.append({"name": name, "M": M, "N": N, "K": K, "transA": ta, "transB": tb, "heuristic_us": heur,
                 "tuned_us": tuned, "cublas_us": cub, "tuned_tflops": fl / tuned / 1e6,
                 "tuned_gbps": byts / tuned / 1e3})
    print(f"{name:18s} M={M:5d} N={N:5d} K={K:5d}  heur {heur:7.2f} us | tuned {tuned:7.2f} us "
          f"{fl / tuned / 1e6:7.1f} TF/s {byts / tuned / 1e3:7.1f} GB/s | cublas {cub:7.2f} us", flush=True)
if out_json:
    with open(out_json, "w") as fh:
        json.dump({"note": f"{R} launches captured in one CUDA graph, replayed; us per launch", "rows": rows},
                  fh, indent=1)
