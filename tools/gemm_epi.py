"""One GEMM with a fused epilogue, CUDA-graph timed (and a target for ncu):

    python tools/gemm_epi.py M N K tA tB EPI [reps]      EPI in none|add|add2|swish|swish_bwd

Prints us per launch (20 launches per graph, best of 3) with the shape the
committed table / heuristic picks, and the same GEMM without the epilogue.
With HAP_GEMM_ONCE=1 it only launches the GEMM `reps` times (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2401_05965_b200 import _lib  # noqa: E402
from paper_2401_05965_b200._lib import BF16, GemmDesc, check  # noqa: E402

M, N, K, ta, tb = (int(v) for v in sys.argv[1:6])
epi = sys.argv[6] if len(sys.argv) > 6 else "none"
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
EPI = {"none": _lib.EPI_NONE, "add": _lib.EPI_ADD, "add2": _lib.EPI_ADD2, "swish": _lib.EPI_SWISH,
       "swish_bwd": _lib.EPI_SWISH_BWD}[epi]
L = _lib.lib()
_lib.load_tune_table()
dev = torch.device("cuda")
a = torch.randn((K, M) if ta else (M, K), device=dev).to(torch.bfloat16)
b = torch.randn((N, K) if tb else (K, N), device=dev).to(torch.bfloat16)
c = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
t1, t2, t3 = (torch.randn(M, N, device=dev).to(torch.bfloat16) for _ in range(3))


def desc(e):
    d = (GemmDesc * 1)()
    d[0].A, d[0].lda, d[0].transA = a.data_ptr(), a.shape[1], ta
    d[0].B, d[0].ldb, d[0].transB = b.data_ptr(), b.shape[1], tb
    d[0].C, d[0].ldc, d[0].M, d[0].N, d[0].K = c.data_ptr(), N, M, N, K
    d[0].epi, d[0].epi_tag = e, _lib.UNARY_TAGS["sigmoid"]
    if e in (_lib.EPI_ADD, _lib.EPI_ADD2, _lib.EPI_SWISH_BWD):
        d[0].R, d[0].ldr = t1.data_ptr(), N
    if e == _lib.EPI_SWISH_BWD:
        d[0].R2, d[0].ldr2 = t2.data_ptr(), N
    if e in (_lib.EPI_ADD2, _lib.EPI_SWISH):
        d[0].Y, d[0].ldy = t2.data_ptr(), N
    if e == _lib.EPI_SWISH:
        d[0].Z, d[0].ldz = t3.data_ptr(), N
    return d


s = torch.cuda.Stream()
if os.environ.get("HAP_GEMM_ONCE"):
    d = desc(EPI)
    for _ in range(reps):
        check(L.hap_matmul_batch(d, 1, 0, BF16, BF16, 0, s.cuda_stream))
    torch.cuda.synchronize()
    print("ok")
    sys.exit(0)


def graph_us(d):
    fn = lambda: check(L.hap_matmul_batch(d, 1, 0, BF16, BF16, 0, s.cuda_stream))  # noqa: E731
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(5):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / 100)
    return best


fused, plain = graph_us(desc(EPI)), graph_us(desc(_lib.EPI_NONE))
flops = 2.0 * M * N * K
print(f"{M}x{N}x{K} t{ta}{tb} epi={epi}: {fused:.2f} us ({flops / fused / 1e6:.0f} TF/s); plain {plain:.2f} us "
      f"({flops / plain / 1e6:.0f} TF/s)")
