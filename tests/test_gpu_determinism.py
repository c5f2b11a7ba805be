"""Run-to-run determinism on the B200: the same inputs give the same bits.

Sources of nondeterminism the executor removes (VERDICT r1 "what's weak" 2):
timing-based tile / split-K choice (now the committed tuning table or the
host heuristic, _lib.load_tune_table), split-K partials combined with
floating-point atomics (now fp32 partial slices summed in split order,
gemm.cu split_reduce_kernel) and cross-CTA reduction atomics (now ticketed ordered sums,
reduce.cu).  Shapes are forced through hap_matmul_tune_import, the same door
the committed table uses."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_2401_05965_b200 import _lib
from paper_2401_05965_b200._lib import BF16, F32, GemmDesc, check

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

L = _lib.lib()
DEV = torch.device("cuda")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _desc(a, ta, b, tb, c, acc=0, epi=_lib.EPI_NONE, R=None, Y=None):
    M, K = (a.shape[1], a.shape[0]) if ta else a.shape
    N = b.shape[0] if tb else b.shape[1]
    d = (GemmDesc * 1)()
    d[0].A, d[0].lda, d[0].transA = a.data_ptr(), a.shape[1], ta
    d[0].B, d[0].ldb, d[0].transB = b.data_ptr(), b.shape[1], tb
    d[0].C, d[0].ldc, d[0].M, d[0].N, d[0].K, d[0].accumulate = c.data_ptr(), c.shape[1], M, N, K, acc
    d[0].epi = epi
    if R is not None:
        d[0].R, d[0].ldr = R.data_ptr(), R.shape[1]
    if Y is not None:
        d[0].Y, d[0].ldy = Y.data_ptr(), Y.shape[1]
    return d


def _key(d, out_f32, cap):
    g = d[0]
    return (f"1/0/{'f' if out_f32 else 'b'}/{cap}|{g.M}x{g.N}x{g.K}:{g.transA}{g.transB}:{g.epi}:{g.accumulate}:"
            f"{g.lda},{g.ldb},{g.ldc}")


def _force(d, out_f32, pair, bn, splits, cap=148):
    kb = (d[0].K + 63) // 64
    kbps = (kb + splits - 1) // splits
    check(L.hap_matmul_tune_import(f"{_key(d, out_f32, cap)}\t{int(pair)} {bn} {splits} {kbps}\n".encode()))


def _run(d, c_dtype, cap=0):
    check(L.hap_matmul_batch(d, 1, 0, BF16, F32 if c_dtype == torch.float32 else BF16, cap, 0), "hap_matmul_batch")
    torch.cuda.synchronize()


@pytest.mark.parametrize("out", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1)])
def test_tile_shape_does_not_change_the_bits(out, ta, tb):
    """Without split K every output element accumulates the same K blocks in
    the same order in TMEM, whatever the tile shape: the table only changes
    speed, never the result."""
    torch.manual_seed(11)
    M, N, K = 1024, 768, 1024
    a = torch.randn((K, M) if ta else (M, K), device=DEV).to(torch.bfloat16)
    b = torch.randn((N, K) if tb else (K, N), device=DEV).to(torch.bfloat16)
    results = []
    try:
        for pair, bn in ((1, 256), (1, 192), (1, 128), (0, 256), (0, 128)):
            c = torch.empty((M, N), device=DEV, dtype=out)
            d = _desc(a, ta, b, tb, c)
            _force(d, out == torch.float32, pair, bn, 1)
            _run(d, out)
            results.append(c.clone())
    finally:
        L.hap_matmul_tune_clear()
    for r in results[1:]:
        assert torch.equal(r, results[0])


@pytest.mark.parametrize("splits", [2, 3, 4, 8])
@pytest.mark.parametrize("pair", [1, 0])
def test_split_k_fp32_accumulate_is_ordered(splits, pair):
    """Weight-gradient shape (fp32 out, accumulate): the K splits' partial
    tiles are summed in split order — 20 eager launches and a CUDA graph
    replay give identical bits, and the result matches fp32 torch."""
    torch.manual_seed(splits)
    M, N, K = 768, 768, 4096
    a = torch.randn(K, M, device=DEV).to(torch.bfloat16)   # A^T . B  (dW = X^T dY)
    b = torch.randn(K, N, device=DEV).to(torch.bfloat16)
    base = torch.randn(M, N, device=DEV)
    c = base.clone()
    d = _desc(a, 1, b, 0, c, acc=1)
    try:
        _force(d, True, pair, 256, splits)
        outs = []
        for _ in range(20):
            c.copy_(base)
            _run(d, torch.float32)
            outs.append(c.clone())
        want = base + a.float().t() @ b.float()
        assert float((outs[0] - want).abs().max() / want.abs().max()) < 1e-5
        for o in outs[1:]:
            assert torch.equal(o, outs[0])
        s = torch.cuda.Stream()
        check(L.hap_matmul_batch(d, 1, 0, BF16, F32, 0, s.cuda_stream))   # eager first: the stream's workspace
        c.copy_(base)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            check(L.hap_matmul_batch(d, 1, 0, BF16, F32, 0, s.cuda_stream))
        for _ in range(3):
            c.copy_(base)
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(c, outs[0])
    finally:
        L.hap_matmul_tune_clear()


@pytest.mark.parametrize("epi", ["none", "add2"])
def test_split_k_bf16_residual_is_ordered(epi):
    """Few-token bf16 GEMM with the residual-add epilogue under split K: the
    ordered reduction applies C = bf16(sum), Y = bf16(bf16(sum) + R)
    identically every run."""
    torch.manual_seed(5)
    M, N, K = 256, 768, 3072
    a = torch.randn(M, K, device=DEV).to(torch.bfloat16)
    b = torch.randn(K, N, device=DEV).to(torch.bfloat16)
    c = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    R = torch.randn(M, N, device=DEV).to(torch.bfloat16)
    Y = torch.empty_like(R)
    d = _desc(a, 0, b, 0, c, epi=_lib.EPI_ADD2 if epi == "add2" else _lib.EPI_NONE,
              R=R if epi == "add2" else None, Y=Y if epi == "add2" else None)
    try:
        _force(d, False, 1, 128, 6)
        outs = []
        for _ in range(20):
            _run(d, torch.bfloat16)
            outs.append((c.clone(), Y.clone()))
        ref = a.float() @ b.float()
        assert float((outs[0][0].float() - ref).abs().max() / ref.abs().max()) < 8e-3
        if epi == "add2":
            want_y = (outs[0][0].float() + R.float()).to(torch.bfloat16)
            assert torch.equal(outs[0][1], want_y)
        for o in outs[1:]:
            assert torch.equal(o[0], outs[0][0]) and (epi != "add2" or torch.equal(o[1], outs[0][1]))
    finally:
        L.hap_matmul_tune_clear()


@pytest.mark.parametrize("shape,dims", [((1 << 23,), (0,)), ((8192, 768), (0,)), ((64, 4096), (1,))])
def test_reductions_are_ordered(shape, dims):
    torch.manual_seed(9)
    x = torch.randn(shape, device=DEV).to(torch.bfloat16)
    out_shape = tuple(e for i, e in enumerate(shape) if i not in dims) or (1,)
    y = torch.empty(out_shape, device=DEV)
    mask = sum(1 << d for d in dims)
    dims_arr = _lib.i64_array(shape)
    outs = []
    for _ in range(30):
        check(L.hap_reduce(x.data_ptr(), BF16, dims_arr, len(shape), mask, y.data_ptr(), F32, 0, 0, 0))
        torch.cuda.synchronize()
        outs.append(y.clone())
    want = x.float().sum(dim=dims).reshape(out_shape)
    assert float((outs[0] - want).abs().max()) <= 1e-4 * max(1.0, float(x.float().abs().sum()) / max(1, want.numel()))
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_two_processes_compute_the_same_bits():
    """Two fresh processes run smoke()'s training iteration (configs[0], two
    devices at 1:2 on SM caps 74/148): identical losses and gradients."""
    code = ("import __graft_entry__ as e; ex, *_ = e._smoke_run(); print('DIGEST', e.smoke_digest(ex))")
    digests = []
    for _ in range(2):
        res = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-3000:]
        digests.append([ln for ln in res.stdout.splitlines() if ln.startswith("DIGEST")][-1])
    assert digests[0] == digests[1], digests
