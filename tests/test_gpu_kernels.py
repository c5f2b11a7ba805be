"""Kernel-level numerics on the B200, through the C ABI, against a plain
PyTorch fp32 reference of the same op (inputs rounded to the kernel's input
precision first).  Tolerances are written per test."""
import numpy as np
import pytest
import torch

from paper_2401_05965_b200 import _lib
from paper_2401_05965_b200._lib import BF16, F32, check

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU collection only
    pytest.skip("needs a GPU", allow_module_level=True)

L = _lib.lib()
DEV = torch.device("cuda")
S = 0  # legacy default stream; tests synchronise explicitly


def _dt(t):
    return BF16 if t.dtype == torch.bfloat16 else F32


def gemm(a, ta, b, tb, c, accumulate=0, sm_cap=0):
    M, K = (a.shape[1], a.shape[0]) if ta else a.shape
    N = b.shape[0] if tb else b.shape[1]
    check(L.hap_matmul(a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb, c.data_ptr(), c.shape[1],
                       M, N, K, _dt(a), _dt(c), accumulate, sm_cap, S), "hap_matmul")
    torch.cuda.synchronize()


def ref_mm(a, ta, b, tb):
    a32, b32 = a.float(), b.float()
    return (a32.t() if ta else a32) @ (b32.t() if tb else b32)


def rel_err(got, want):
    return float((got.float() - want).abs().max() / max(want.abs().max().item(), 1e-6))


SHAPES = [(128, 128, 64), (256, 512, 320), (300, 200, 72), (1000, 520, 1000), (64, 1024, 1024),
          (4096, 3072, 768), (8, 264, 40), (8192, 768, 3072), (2048, 768, 1024)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("out", [torch.bfloat16, torch.float32])
def test_tcgen05_gemm_all_orientations(M, N, K, ta, tb, out):
    torch.manual_seed(M * 7 + N * 3 + K + ta * 2 + tb)
    a = torch.randn((K, M) if ta else (M, K), device=DEV).to(torch.bfloat16)
    b = torch.randn((N, K) if tb else (K, N), device=DEV).to(torch.bfloat16)
    # tcgen05 needs 16-byte row pitches (TMA); other shapes take the SIMT kernel.
    tma_ok = a.shape[1] % 8 == 0 and b.shape[1] % 8 == 0
    engine = L.hap_matmul_engine(a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb, M, N, K, BF16)
    assert engine == (_lib.GEMM_TCGEN05 if tma_ok else _lib.GEMM_SIMT)
    c = torch.empty((M, N), device=DEV, dtype=out)
    gemm(a, ta, b, tb, c)
    want = ref_mm(a, ta, b, tb)
    # fp32 accumulate in TMEM: only summation order differs (fp32 out), plus
    # one bf16 rounding of the result (bf16 out).
    assert rel_err(c, want) < (1e-5 if out == torch.float32 else 8e-3)


def test_gemm_accumulate_and_sm_cap():
    torch.manual_seed(1)
    a = torch.randn(512, 256, device=DEV).to(torch.bfloat16)
    b = torch.randn(256, 384, device=DEV).to(torch.bfloat16)
    c = torch.randn(512, 384, device=DEV)
    base = c.clone()
    gemm(a, 0, b, 0, c, accumulate=1, sm_cap=7)
    assert rel_err(c, base + ref_mm(a, 0, b, 0)) < 1e-5


@pytest.mark.parametrize("M,N,K", [(8, 2, 4), (6, 2, 4), (0, 4, 4), (5, 0, 3), (3, 3, 0), (33, 17, 9)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_simt_gemm_small_and_zero_shapes(M, N, K, dtype):
    torch.manual_seed(2)
    for ta, tb in [(0, 0), (1, 0), (0, 1)]:
        a = torch.randn((K, M) if ta else (M, K), device=DEV).to(dtype)
        b = torch.randn((N, K) if tb else (K, N), device=DEV).to(dtype)
        c = torch.full((M, N), 7.0, device=DEV)
        if M and N:
            gemm(a, ta, b, tb, c)
            want = ref_mm(a, ta, b, tb)
            assert rel_err(c, want) < 1e-5 or want.abs().max() == 0


@pytest.mark.parametrize("tag", ["exp", "neg", "relu", "sigmoid", "tanh"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_unary_and_adjoint(tag, dtype):
    torch.manual_seed(3)
    n = 100003
    x = torch.randn(n, device=DEV).to(dtype)
    y = torch.empty_like(x)
    check(L.hap_unary(_lib.UNARY_TAGS[tag], x.data_ptr(), _dt(x), y.data_ptr(), _dt(y), n, 0, S))
    xf = x.float()
    fn = {"exp": torch.exp, "neg": torch.neg, "relu": torch.relu, "sigmoid": torch.sigmoid, "tanh": torch.tanh}[tag]
    tol = 1e-5 if dtype == torch.float32 else 8e-3
    torch.cuda.synchronize()
    assert rel_err(y, fn(xf)) < tol
    dy = torch.randn(n, device=DEV).to(dtype)
    dx = torch.full((n,), 1.0, device=DEV)
    check(L.hap_unary_grad(_lib.UNARY_TAGS[tag], x.data_ptr(), y.data_ptr(), _dt(x), dy.data_ptr(), _dt(dy),
                           dx.data_ptr(), F32, n, 1, 0, S))
    xr = xf.clone().requires_grad_(True)
    fn(xr).backward(dy.float())
    torch.cuda.synchronize()
    assert rel_err(dx, 1.0 + xr.grad) < (1e-4 if dtype == torch.float32 else 2e-2)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_binary_and_mul_adjoint(dtype):
    torch.manual_seed(4)
    n = 65537
    a, b = torch.randn(n, device=DEV).to(dtype), torch.randn(n, device=DEV).to(dtype)
    for tag, fn in (("add", torch.add), ("mul", torch.mul)):
        out = torch.empty(n, device=DEV)
        check(L.hap_binary(_lib.BINARY_TAGS[tag], a.data_ptr(), b.data_ptr(), _dt(a), out.data_ptr(), F32, n, 0, S))
        torch.cuda.synchronize()
        assert rel_err(out, fn(a.float(), b.float())) < 1e-6
    dy = torch.randn(n, device=DEV)
    da, db = torch.zeros(n, device=DEV), torch.zeros(n, device=DEV)
    check(L.hap_mul_grad(a.data_ptr(), b.data_ptr(), _dt(a), dy.data_ptr(), F32, da.data_ptr(), db.data_ptr(),
                         F32, n, 0, 0, S))
    torch.cuda.synchronize()
    assert rel_err(da, dy * b.float()) < 1e-6 and rel_err(db, dy * a.float()) < 1e-6
    # self-product: d(a*a)/da = 2a
    check(L.hap_mul_grad(a.data_ptr(), a.data_ptr(), _dt(a), dy.data_ptr(), F32, da.data_ptr(), da.data_ptr(),
                         F32, n, 0, 0, S))
    torch.cuda.synchronize()
    assert rel_err(da, 2 * dy * a.float()) < 1e-6


@pytest.mark.parametrize("shape,dims", [((8192, 768), (0, 1)), ((8192, 768), (0,)), ((8192, 768), (1,)),
                                        ((5, 7), (1,)), ((3, 4, 5), (0, 2)), ((3, 4, 5), (1,)),
                                        ((6, 0), (0,)), ((16,), (0,)), ((2, 3, 4, 5), (1, 2))])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_reduce_and_unreduce(shape, dims, dtype):
    torch.manual_seed(5)
    x = torch.randn(shape, device=DEV).to(dtype)
    out_shape = tuple(e for a, e in enumerate(shape) if a not in dims)
    y = torch.full(out_shape, 3.0, device=DEV)
    mask = sum(1 << d for d in dims)
    shp = _lib.i64_array(shape)
    check(L.hap_reduce(x.data_ptr(), _dt(x), shp, len(shape), mask, y.data_ptr(), F32, 0, 0, S))
    torch.cuda.synchronize()
    want = x.float().sum(dim=dims)
    if want.numel() == 0:
        return
    assert (y - want).abs().max().item() <= 1e-4 * max(1.0, x.float().abs().sum().item() / max(1, want.numel()))
    dy = torch.randn(out_shape, device=DEV)
    dx = torch.ones(shape, device=DEV)
    check(L.hap_unreduce(dy.data_ptr(), F32, shp, len(shape), mask, dx.data_ptr(), F32, 1, 0, S))
    torch.cuda.synchronize()
    expand = dy
    for d in sorted(dims):
        expand = expand.unsqueeze(d)
    assert torch.allclose(dx, 1.0 + expand.expand(shape))


def test_copy_block_strided_shards():
    torch.manual_seed(6)
    src = torch.randn(6, 10, 3, device=DEV)
    dst = torch.zeros(6, 4, 3, device=DEV, dtype=torch.bfloat16)
    check(L.hap_copy_block(src.data_ptr(), F32, 10, 5, dst.data_ptr(), BF16, 4, 1, 6, 3, 3, 0, 0, S))
    torch.cuda.synchronize()
    assert torch.equal(dst[:, 1:4].float(), src[:, 5:8].to(torch.bfloat16).float())
    assert dst[:, 0].abs().max().item() == 0


def test_sgd_multi_tensor():
    import struct
    torch.manual_seed(7)
    sizes = [1000, 8192 * 3 + 5, 16, 70000]
    masters = [torch.randn(n, device=DEV) for n in sizes]
    grads = [torch.randn(n, device=DEV) for n in sizes]
    weights = [torch.empty(n, device=DEV, dtype=torch.bfloat16) for n in sizes]
    want = [m - 0.5 * g for m, g in zip(masters, grads)]
    rec, chunk = bytearray(), 0
    for m, g, w in zip(masters, grads, weights):
        rec += struct.pack("<QQQqq", m.data_ptr(), g.data_ptr(), w.data_ptr(), m.numel(), chunk)
        chunk += (m.numel() + 8191) // 8192
    table = torch.frombuffer(bytes(rec), dtype=torch.uint8).to(DEV)
    check(L.hap_sgd_multi(table.data_ptr(), len(sizes), chunk, BF16, 0.5, 0, S))
    torch.cuda.synchronize()
    for m, w, ref in zip(masters, weights, want):
        assert torch.allclose(m, ref) and torch.equal(w, ref.to(torch.bfloat16))


def _desc(a, ta, b, tb, c, acc=0):
    M, K = (a.shape[1], a.shape[0]) if ta else a.shape
    N = b.shape[0] if tb else b.shape[1]
    return _lib.GemmDesc(a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb, c.data_ptr(), c.shape[1],
                         M, N, K, acc)


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0)])
@pytest.mark.parametrize("out", [torch.bfloat16, torch.float32])
def test_matmul_batch_grouped_and_summed(ta, tb, out):
    torch.manual_seed(11)
    M, N, K = 1024, 768, 512
    mk = lambda r, c: torch.randn(r, c, device=DEV).to(torch.bfloat16)  # noqa: E731
    # grouped: three independent problems sharing A
    a = mk(K, M) if ta else mk(M, K)
    bs = [mk(N, K) if tb else mk(K, N) for _ in range(3)]
    cs = [torch.empty(M, N, device=DEV, dtype=out) for _ in range(3)]
    descs = (_lib.GemmDesc * 3)(*[_desc(a, ta, b, tb, c) for b, c in zip(bs, cs)])
    check(L.hap_matmul_batch(descs, 3, 0, BF16, _dt(cs[0]), 0, S))
    torch.cuda.synchronize()
    tol = 1e-5 if out == torch.float32 else 8e-3
    for b, c in zip(bs, cs):
        assert rel_err(c, ref_mm(a, ta, b, tb)) < tol
    # summed: C = sum_i A_i . B_i (+ C), five problems (chunked 4 + 1)
    As = [mk(K, M) if ta else mk(M, K) for _ in range(5)]
    Bs = [mk(N, K) if tb else mk(K, N) for _ in range(5)]
    c = torch.randn(M, N, device=DEV).to(out)
    base = c.float().clone()
    descs = (_lib.GemmDesc * 5)(*[_desc(x, ta, y, tb, c, acc=1) for x, y in zip(As, Bs)])
    check(L.hap_matmul_batch(descs, 5, 1, BF16, _dt(c), 0, S))
    torch.cuda.synchronize()
    want = base + sum(ref_mm(x, ta, y, tb) for x, y in zip(As, Bs))
    assert rel_err(c, want) < (1e-5 if out == torch.float32 else 1.2e-2)


@pytest.mark.parametrize("M,N,K", [(256, 768, 3072), (256, 3072, 768), (200, 520, 4096), (128, 96, 2048),
                                   (512, 1000, 1536)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0)])
@pytest.mark.parametrize("acc", [0, 1])
def test_split_k_into_bf16_output(M, N, K, ta, tb, acc):
    """Few output tiles, long K: the K range is split across SMs, partial sums
    meet in the fp32 workspace and the last split rounds them into the bf16
    output.  Repeated launches check that the workspace and its counters are
    left clean; a capped grid checks the persistent schedule."""
    torch.manual_seed(M + N + K + ta + tb + acc)
    a = torch.randn((K, M) if ta else (M, K), device=DEV).to(torch.bfloat16)
    b = torch.randn((N, K) if tb else (K, N), device=DEV).to(torch.bfloat16)
    want = ref_mm(a, ta, b, tb)
    for cap in (0, 0, 23):
        c = torch.randn(M, N, device=DEV).to(torch.bfloat16)
        base = c.float().clone()
        gemm(a, ta, b, tb, c, accumulate=acc, sm_cap=cap)
        assert rel_err(c, want + base if acc else want) < 8e-3, cap


def test_split_k_bf16_sum_and_graph_replay():
    """A K-concatenated sum (dx = dq.Wq^T + dk.Wk^T + dv.Wv^T at few tokens)
    splits its combined K range; the same launches replay from a CUDA graph."""
    torch.manual_seed(5)
    M, N, K = 256, 768, 768
    As = [torch.randn(M, K, device=DEV).to(torch.bfloat16) for _ in range(3)]
    Bs = [torch.randn(N, K, device=DEV).to(torch.bfloat16) for _ in range(3)]
    c = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    descs = (_lib.GemmDesc * 3)(*[_desc(x, 0, y, 1, c) for x, y in zip(As, Bs)])
    want = sum(ref_mm(x, 0, y, 1) for x, y in zip(As, Bs))
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        check(L.hap_matmul_batch(descs, 3, 1, BF16, BF16, 0, stream.cuda_stream))
    stream.synchronize()
    assert rel_err(c, want) < 8e-3
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        check(L.hap_matmul_batch(descs, 3, 1, BF16, BF16, 0, stream.cuda_stream))
    for _ in range(3):
        c.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert rel_err(c, want) < 8e-3


@pytest.mark.parametrize("cap", [0, 8])
@pytest.mark.parametrize("out", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("K", [256, 200, 4096])
def test_matmul_batch_grouped_mixed_shapes(out, K, cap):
    """Grouped problems of different M x N in one launch (the weight
    gradients of a layer rebuilt from gathered factors: dW = X^T . dY).  A
    small SM cap makes every CTA drain many tiles in a row (epilogue staging
    buffers alternate across tiles with an odd box count, 192-wide tiles)."""
    torch.manual_seed(K)
    shapes = [(3072, 768), (768, 3072), (768, 768), (768, 768)]
    As = [torch.randn(K, M, device=DEV).to(torch.bfloat16) for M, _ in shapes]
    Bs = [torch.randn(K, N, device=DEV).to(torch.bfloat16) for _, N in shapes]
    Cs = [torch.full((M, N), 7.0, device=DEV, dtype=out) for M, N in shapes]
    descs = (_lib.GemmDesc * 4)(*[_desc(a, 1, b, 0, c) for a, b, c in zip(As, Bs, Cs)])
    check(L.hap_matmul_batch(descs, 4, 0, BF16, _dt(Cs[0]), cap, S))
    torch.cuda.synchronize()
    for a, b, c in zip(As, Bs, Cs):
        assert rel_err(c, ref_mm(a, 1, b, 0)) < (1e-5 if out == torch.float32 else 8e-3)


def _fdesc(a, ta, b, tb, c, accumulate=0, **epi):
    M, K = (a.shape[1], a.shape[0]) if ta else a.shape
    N = b.shape[0] if tb else b.shape[1]
    d = _lib.GemmDesc()
    d.A, d.lda, d.transA, d.B, d.ldb, d.transB = a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb
    d.C, d.ldc, d.M, d.N, d.K, d.accumulate = c.data_ptr(), c.shape[1], M, N, K, accumulate
    fields = {f for f, _ in _lib.GemmDesc._fields_}
    for k, v in epi.items():
        assert k in fields, k
        setattr(d, k, v.data_ptr() if isinstance(v, torch.Tensor) else v)
    for k, ld in (("R", "ldr"), ("R2", "ldr2"), ("Y", "ldy"), ("Z", "ldz")):
        if isinstance(epi.get(k), torch.Tensor):
            setattr(d, ld, epi[k].shape[1])
    return d


def _run_descs(descs, out_dt=BF16, sum_k=0, sm_cap=0):
    arr = (_lib.GemmDesc * len(descs))(*descs)
    check(L.hap_matmul_batch(arr, len(descs), sum_k, BF16, out_dt, sm_cap, S), "hap_matmul_batch")
    torch.cuda.synchronize()


def _bf(t):
    return t.to(torch.bfloat16).float()


# (256, 768, 3072): few tiles and 48 K blocks — split K, the residual
# epilogues (add, add_self, add2) run in the split reduction
SPLIT_EPI_SHAPE = (256, 768, 3072)
EPI_SHAPES = [(8192, 768, 3072), (1000, 520, 200), (256, 3072, 768), (300, 136, 64), SPLIT_EPI_SHAPE]


@pytest.mark.parametrize("M,N,K", EPI_SHAPES)
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0)])
@pytest.mark.parametrize("epi", ["add", "add_self", "add2", "swish", "swish_bwd", "swish_bwd_acc"])
def test_gemm_fused_epilogues(M, N, K, ta, tb, epi):
    """Fused epilogues (hap_gemm_desc.epi) against the unfused sequence of
    our own kernels (GEMM into bf16, then the elementwise kernel) — the same
    roundings, so equal up to fp32 contraction differences (<= 1 bf16 ulp on
    a few elements) — and against a PyTorch fp32 reference (2e-2)."""
    if (M, N, K) == SPLIT_EPI_SHAPE and epi.startswith("swish"):
        # the swish chains never split K, the plain GEMM they are compared
        # with does at this shape: summation orders differ by design
        pytest.skip("swish epilogues do not split K")
    torch.manual_seed(M + 3 * N + 7 * K + ta + 2 * tb)
    a = torch.randn((K, M) if ta else (M, K), device=DEV).to(torch.bfloat16)
    b = (torch.randn((N, K) if tb else (K, N), device=DEV) / K ** 0.5).to(torch.bfloat16)
    mm = ref_mm(a, ta, b, tb)
    c = torch.empty((M, N), device=DEV, dtype=torch.bfloat16)
    r = torch.randn((M, N), device=DEV).to(torch.bfloat16)
    sig = _lib.UNARY_TAGS["sigmoid"]
    if L.hap_matmul_engine(a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb, M, N, K,
                           BF16) != _lib.GEMM_TCGEN05:
        # fused epilogues exist on the tcgen05 path only: loud error, no silent fallback
        with pytest.raises(_lib.HapError, match="fused epilogues"):
            _run_descs([_fdesc(a, ta, b, tb, c, epi=_lib.EPI_ADD, R=r)])
        return
    plain = torch.empty_like(c)
    gemm(a, ta, b, tb, plain)
    n = M * N
    if epi == "add":
        _run_descs([_fdesc(a, ta, b, tb, c, epi=_lib.EPI_ADD, R=r)])
        want, fused, unfused = mm + r.float(), [c], None
    elif epi == "add_self":
        c.copy_(r)
        _run_descs([_fdesc(a, ta, b, tb, c, accumulate=1, epi=_lib.EPI_ADD)])
        want, fused, unfused = mm + r.float(), [c], None
    elif epi == "add2":
        y = torch.empty_like(c)
        _run_descs([_fdesc(a, ta, b, tb, c, epi=_lib.EPI_ADD2, R=r, Y=y)])
        y2 = torch.empty_like(c)
        check(L.hap_binary(_lib.BINARY_TAGS["add"], plain.data_ptr(), r.data_ptr(), BF16, y2.data_ptr(), BF16, n,
                           0, S), "hap_binary")
        want, fused, unfused = _bf(mm) + r.float(), [c, y], [plain, y2]
    elif epi == "swish":
        y, z = torch.empty_like(c), torch.empty_like(c)
        _run_descs([_fdesc(a, ta, b, tb, c, epi=_lib.EPI_SWISH, epi_tag=sig, Y=y, Z=z)])
        y2, z2 = torch.empty_like(c), torch.empty_like(c)
        check(L.hap_swish_fwd(sig, plain.data_ptr(), y2.data_ptr(), z2.data_ptr(), BF16, n, 0, S), "hap_swish_fwd")
        s = torch.sigmoid(_bf(mm))
        want, fused, unfused = _bf(mm) * _bf(s), [c, y, z], [plain, y2, z2]
        assert rel_err(y, s) < 2e-2
    elif epi == "swish_bwd_acc":
        # the fused adjoint writes its output (no read-modify-write): loud error
        x = torch.randn((M, N), device=DEV).to(torch.bfloat16)
        with pytest.raises(_lib.HapError, match="no accumulate"):
            _run_descs([_fdesc(a, ta, b, tb, c, accumulate=1, epi=_lib.EPI_SWISH_BWD, epi_tag=sig, R=x, R2=x)])
        return
    else:
        acc = False
        x = torch.randn((M, N), device=DEV).to(torch.bfloat16)
        xs = torch.sigmoid(x.float()).to(torch.bfloat16)
        dx = torch.randn((M, N), device=DEV).to(torch.bfloat16) if acc else torch.empty_like(c)
        dx2 = dx.clone()
        _run_descs([_fdesc(a, ta, b, tb, dx, accumulate=int(acc), epi=_lib.EPI_SWISH_BWD, epi_tag=sig, R=x, R2=xs)])
        check(L.hap_swish_bwd(sig, x.data_ptr(), xs.data_ptr(), plain.data_ptr(), dx2.data_ptr(), BF16, n,
                              int(acc), 0, S), "hap_swish_bwd")
        g, xf, yf = _bf(mm), x.float(), xs.float()
        want = g * yf + g * xf * yf * (1 - yf) + (dx2.float() * 0 if not acc else 0)
        fused, unfused = [dx], [dx2]
        if acc:
            want = None   # checked against the unfused kernels only
    torch.cuda.synchronize()
    if unfused is not None:
        for f, u in zip(fused, unfused):
            diff = (f.float() - u.float()).abs()
            ulp = u.float().abs().clamp_min(1e-30) * 2.0 ** -7
            assert int((diff > ulp).sum()) == 0, (epi, float(diff.max()))
            assert float((diff > 0).float().mean()) < 1e-3, (epi, float((diff > 0).float().mean()))
    if want is not None:
        assert rel_err(fused[-1], want) < 2e-2


@pytest.mark.parametrize("cap", [0, 104, 88, 20])
@pytest.mark.parametrize("M,N,K", [(8192, 768, 3072), (8192, 3072, 1536), (2048, 1000, 1040)])
def test_stream_k_gemm_repeated_and_graph(M, N, K, cap, monkeypatch):
    """Shapes whose data-parallel rounds leave SM pairs idle run stream-K
    (equal K-block ranges per pair, cut tiles finished from an fp32 partial):
    results match the fp32 reference, stay identical over repeated launches
    (the partial flags reset themselves) and under CUDA-graph replay."""
    monkeypatch.setenv("HAP_GEMM_SK", "1")   # opt-in path (off by default)
    torch.manual_seed(M + N + K + cap)
    a = torch.randn(M, K, device=DEV).to(torch.bfloat16)
    b = (torch.randn(K, N, device=DEV) / K ** 0.5).to(torch.bfloat16)
    r = torch.randn(M, N, device=DEV).to(torch.bfloat16)
    want = ref_mm(a, 0, b, 0)
    outs = []
    for _ in range(3):
        c = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
        gemm(a, 0, b, 0, c, sm_cap=cap)
        outs.append(c)
    assert rel_err(outs[0], want) < 8e-3
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    y = torch.empty_like(r)
    c = torch.empty_like(r)
    _run_descs([_fdesc(a, 0, b, 0, c, epi=_lib.EPI_ADD2, R=r, Y=y)], sm_cap=cap)
    assert torch.equal(c, outs[0])
    assert rel_err(y, want + r.float()) < 2e-2
    # graph replay on a side stream
    s = torch.cuda.Stream()
    cg = torch.zeros(M, N, device=DEV, dtype=torch.bfloat16)
    with torch.cuda.stream(s):
        check(L.hap_matmul(a.data_ptr(), K, 0, b.data_ptr(), N, 0, cg.data_ptr(), N, M, N, K, BF16, BF16, 0, cap,
                           s.cuda_stream), "warm")
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        check(L.hap_matmul(a.data_ptr(), K, 0, b.data_ptr(), N, 0, cg.data_ptr(), N, M, N, K, BF16, BF16, 0, cap,
                           s.cuda_stream), "capture")
    for _ in range(3):
        cg.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(cg, outs[0])


@pytest.mark.parametrize("case", ["bf16", "f32_acc", "add_acc", "sum_k", "swish"])
def test_matmul_tune_keeps_outputs_and_results(case):
    """hap_matmul_tune times candidate shapes on scratch outputs: the real
    outputs are untouched by tuning, and launches after tuning (with the
    chosen shape) still match the fp32 reference."""
    torch.manual_seed(5)
    M, N, K = 4096, 1536, 1024
    a = torch.randn(M, K, device=DEV).to(torch.bfloat16)
    b = (torch.randn(K, N, device=DEV) / K ** 0.5).to(torch.bfloat16)
    want = ref_mm(a, 0, b, 0)
    out_dt = F32 if case == "f32_acc" else BF16
    c = torch.randn(M, N, device=DEV).to(torch.float32 if case == "f32_acc" else torch.bfloat16)
    base = c.clone()
    if case == "bf16":
        descs = [_fdesc(a, 0, b, 0, c)]
    elif case in ("f32_acc", "add_acc"):
        descs = [_fdesc(a, 0, b, 0, c, accumulate=1, **({"epi": _lib.EPI_ADD} if case == "add_acc" else {}))]
        want = want + base.float()
    elif case == "sum_k":
        a2 = torch.randn(M, K, device=DEV).to(torch.bfloat16)
        descs = [_fdesc(a, 0, b, 0, c), _fdesc(a2, 0, b, 0, c, accumulate=1)]
        want = want + ref_mm(a2, 0, b, 0)
    else:
        y, z = torch.empty_like(c), torch.empty_like(c)
        descs = [_fdesc(a, 0, b, 0, c, epi=_lib.EPI_SWISH, epi_tag=_lib.UNARY_TAGS["sigmoid"], Y=y, Z=z)]
    arr = (_lib.GemmDesc * len(descs))(*descs)
    check(L.hap_matmul_tune(arr, len(descs), int(case == "sum_k"), BF16, out_dt, 0, S), "hap_matmul_tune")
    torch.cuda.synchronize()
    assert torch.equal(c, base)   # tuning wrote only scratch
    check(L.hap_matmul_batch(arr, len(descs), int(case == "sum_k"), BF16, out_dt, 0, S), "hap_matmul_batch")
    torch.cuda.synchronize()
    assert rel_err(c, want) < (1e-5 if case == "f32_acc" else 1.2e-2)


@pytest.mark.gpu
@pytest.mark.parametrize("tune", [0, 1])
def test_split_k_residual_epilogue_sum_and_graph(tune):
    """The MoE backward's dx = dy0.W0^T + dy1.W1^T + R (K-concatenated sum with
    a fused residual addend, 96 K blocks over 3-12 output tiles) splits K; the
    split reduction adds R.  Against fp32 torch, and repeated / graph-replayed
    launches give identical bits (ordered reduction)."""
    torch.manual_seed(11)
    M, N, K = 256, 768, 3072
    a0, a1 = (torch.randn(M, K, device=DEV).to(torch.bfloat16) for _ in range(2))
    w0, w1 = ((torch.randn(N, K, device=DEV) / K ** 0.5).to(torch.bfloat16) for _ in range(2))
    r = torch.randn(M, N, device=DEV).to(torch.bfloat16)
    c = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    arr = (_lib.GemmDesc * 2)(_fdesc(a0, 0, w0, 1, c, epi=_lib.EPI_ADD, R=r), _fdesc(a1, 0, w1, 1, c, accumulate=1))
    s = torch.cuda.Stream()
    run = lambda: check(L.hap_matmul_batch(arr, 2, 1, BF16, BF16, 0, s.cuda_stream), "hap_matmul_batch")
    with torch.cuda.stream(s):
        if tune:
            check(L.hap_matmul_tune(arr, 2, 1, BF16, BF16, 0, s.cuda_stream), "hap_matmul_tune")
        run()
    torch.cuda.synchronize()
    want = a0.float() @ w0.float().t() + a1.float() @ w1.float().t() + r.float()
    assert rel_err(c, want) < 2e-2
    first = c.clone()
    with torch.cuda.stream(s):
        run()
    torch.cuda.synchronize()
    assert torch.equal(c, first)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        run()
    c.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(c, first)
