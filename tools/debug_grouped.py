import sys, torch
sys.path.insert(0, ".")
from paper_2401_05965_b200 import _lib
from paper_2401_05965_b200._lib import BF16, F32, check
L = _lib.lib(); DEV = torch.device("cuda")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
shapes = [tuple(int(v) for v in s.split("x")) for s in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["3072x768", "768x3072", "768x768", "768x768"])]
out = torch.float32
torch.manual_seed(0)
As = [torch.randn(K, M, device=DEV).to(torch.bfloat16) for M, _ in shapes]
Bs = [torch.randn(K, N, device=DEV).to(torch.bfloat16) for _, N in shapes]
Cs = [torch.full((M, N), 7.0, device=DEV, dtype=out) for M, N in shapes]
descs = (_lib.GemmDesc * len(shapes))(*[_lib.GemmDesc(a.data_ptr(), a.shape[1], 1, b.data_ptr(), b.shape[1], 0, c.data_ptr(), c.shape[1], c.shape[0], c.shape[1], K, 0) for a, b, c in zip(As, Bs, Cs)])
check(L.hap_matmul_batch(descs, len(shapes), 0, BF16, F32, 0, 0))
torch.cuda.synchronize()
for q, (a, b, c) in enumerate(zip(As, Bs, Cs)):
    want = a.float().t() @ b.float()
    bad = (c - want).abs() > 1e-3 * want.abs().max()
    print(q, c.shape, "bad", int(bad.sum()), "of", bad.numel())
    if bad.any():
        rows = bad.any(1).nonzero().flatten(); cols = bad.any(0).nonzero().flatten()
        print("   rows", rows.min().item(), rows.max().item(), "cols", cols.min().item(), cols.max().item())
        tb = bad.reshape(c.shape[0] // 128, 128, c.shape[1] // 128, 128).any(3).any(1)
        print("   bad 128x128 blocks:", tb.nonzero().tolist()[:20])
        print("   sample got", c[rows[0], cols[0]].item(), "want", want[rows[0], cols[0]].item())
