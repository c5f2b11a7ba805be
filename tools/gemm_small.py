"""Back-to-back launch time of small GEMM shapes (CUDA events, L2-warm):
python tools/gemm_small.py [reps]   — environment toggles (HAP_GEMM_PAIR,
HAP_GEMM_SPLIT) select the variants to compare."""
import sys

import torch

sys.path.insert(0, ".")  # package of the current directory
from paper_2401_05965_b200 import _lib  # noqa: E402
from paper_2401_05965_b200._lib import BF16, F32, check  # noqa: E402

SHAPES = [  # M, N, K, ta, tb, out
    (256, 768, 3072, 0, 0, "bf16"), (256, 768, 3072, 0, 1, "bf16"), (256, 3072, 768, 0, 0, "bf16"),
    (256, 3072, 768, 0, 1, "bf16"), (768, 3072, 256, 1, 0, "f32"), (3072, 768, 256, 1, 0, "f32"),
    (8192, 768, 768, 0, 0, "bf16"), (8192, 3072, 768, 0, 0, "bf16"), (8192, 768, 3072, 0, 0, "bf16"),
    (768, 768, 8192, 1, 0, "f32"), (128, 128, 64, 0, 0, "bf16"),
]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
L = _lib.lib()
dev = torch.device("cuda")
for M, N, K, ta, tb, out in SHAPES:
    a = torch.randn((K, M) if ta else (M, K), device=dev).to(torch.bfloat16)
    b = torch.randn((N, K) if tb else (K, N), device=dev).to(torch.bfloat16)
    c = torch.empty((M, N), device=dev, dtype=torch.float32 if out == "f32" else torch.bfloat16)
    odt = F32 if out == "f32" else BF16

    def run():
        check(L.hap_matmul(a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb, c.data_ptr(), N, M, N, K,
                           BF16, odt, 0, 0, torch.cuda.current_stream().cuda_stream))
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):   # warm on the capture stream (its split-K workspace)
        for _ in range(5):
            run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(20):
            run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps // 20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / (reps // 20 * 20) * 1e3
    print(f"M={M:5d} N={N:5d} K={K:5d} tA={ta} tB={tb} {out:4s} {us:8.2f} us  {2 * M * N * K / us / 1e6:7.1f} TF/s",
          flush=True)
