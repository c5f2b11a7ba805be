"""Split-K A/B on the few-tile GEMM shapes (suffix c: cluster split K, DSMEM
reduction; no suffix: workspace slices + ordered reduction kernel) (MoE 256-token stack, BERT weight
gradients): every tile shape x split candidate forced through the tuning
table, CUDA-graph timed (20 launches per graph).  With --lib PATH a second
build (e.g. the round-1 library, abtest/libgemm_r01.so) is timed the same
way after its own hap_matmul_tune pick.

    python tools/split_bench.py [--lib abtest/libgemm_r01.so]
"""
import argparse
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2401_05965_b200 import _lib  # noqa: E402
from paper_2401_05965_b200._lib import BF16, F32, GemmDesc  # noqa: E402

SHAPES = [  # name, M, N, K, transA, transB, out, accumulate, epi
    ("moe f1", 256, 3072, 768, 0, 0, "bf16", 0, 0),
    ("moe y +res", 256, 768, 3072, 0, 0, "bf16", 0, 2),
    ("moe dx", 256, 768, 3072, 0, 1, "bf16", 0, 0),
    ("moe dW1", 768, 3072, 256, 1, 0, "f32", 1, 0),
    ("moe dW2", 3072, 768, 256, 1, 0, "f32", 1, 0),
    ("bert dWo", 768, 768, 8192, 1, 0, "f32", 1, 0),
    ("bert dW1", 768, 3072, 8192, 1, 0, "f32", 1, 0),
]


def graph_us(fn, stream, reps=20, iters=10):
    with torch.cuda.stream(stream):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(iters):
                g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / (iters * reps))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    args = ap.parse_args()
    L = _lib.lib()
    other = None
    if args.lib:
        other = ctypes.CDLL(args.lib)
        other.hap_matmul_batch.argtypes = [ctypes.POINTER(GemmDesc), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        other.hap_matmul_tune.argtypes = other.hap_matmul_batch.argtypes
    dev = torch.device("cuda")
    s = torch.cuda.Stream()
    for name, M, N, K, ta, tb, out, acc, epi in SHAPES:
        a = torch.randn((K, M) if ta else (M, K), device=dev).to(torch.bfloat16)
        b = torch.randn((N, K) if tb else (K, N), device=dev).to(torch.bfloat16)
        c = torch.zeros((M, N), device=dev, dtype=torch.float32 if out == "f32" else torch.bfloat16)
        R = torch.randn(M, N, device=dev).to(torch.bfloat16)
        Y = torch.empty_like(R)
        d = (GemmDesc * 1)()
        d[0].A, d[0].lda, d[0].transA = a.data_ptr(), a.shape[1], ta
        d[0].B, d[0].ldb, d[0].transB = b.data_ptr(), b.shape[1], tb
        d[0].C, d[0].ldc, d[0].M, d[0].N, d[0].K = c.data_ptr(), N, M, N, K
        d[0].accumulate, d[0].epi = acc, epi
        if epi:
            d[0].R, d[0].ldr, d[0].Y, d[0].ldy = R.data_ptr(), N, Y.data_ptr(), N
        odt = F32 if out == "f32" else BF16
        key = f"1/0/{'f' if out == 'f32' else 'b'}/148|{M}x{N}x{K}:{ta}{tb}:{epi}:{acc}:{d[0].lda},{d[0].ldb},{N}"
        kb = (K + 63) // 64
        res = []
        for pair, bn in ((1, 256), (1, 192), (1, 128), (0, 256), (0, 128)):
            rows = 256 if pair else 128
            if pair and M < 256:
                continue
            tiles = -(-M // rows) * -(-N // bn)
            slots = 74 if pair else 148
            for sp in (1, 2, 3, 4, 6, 8, 12, 16):
                if sp > 1 and (tiles * sp > slots or kb // sp < 2):
                    continue
                kbps = -(-kb // sp)
                for cl in ((0, 1) if (sp in (2, 4) or (sp == 8 and not pair)) else (0,)):
                    L.hap_matmul_tune_import(f"{key}\t{pair} {bn} {sp} {kbps} {cl}\n".encode())
                    us = graph_us(lambda: L.hap_matmul_batch(d, 1, 0, BF16, odt, 0, s.cuda_stream), s)
                    res.append((us, f"{'pair' if pair else 'cta'}{bn}/s{sp}{'c' if cl else ''}"))
        L.hap_matmul_tune_clear()
        res.sort()
        heur = graph_us(lambda: L.hap_matmul_batch(d, 1, 0, BF16, odt, 0, s.cuda_stream), s)
        line = (f"{name:12s} {M}x{N}x{K}: best {res[0][1]} {res[0][0]:.2f} us; heuristic {heur:.2f} us; "
                + " ".join(f"{n}={u:.1f}" for u, n in res[:8]))
        if other is not None:
            other.hap_matmul_tune(d, 1, 0, BF16, odt, 0, s.cuda_stream)
            old = graph_us(lambda: other.hap_matmul_batch(d, 1, 0, BF16, odt, 0, s.cuda_stream), s)
            line += f"; r01 tuned {old:.2f} us"
        print(line, flush=True)


if __name__ == "__main__":
    main()
