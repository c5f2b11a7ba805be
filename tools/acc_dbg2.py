import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import test_gpu_kernels as T
from paper_2401_05965_b200 import _lib
from paper_2401_05965_b200._lib import BF16, check
DEV = torch.device("cuda")
torch.manual_seed(11)
M, N, K = 1024, 768, 512
mk = lambda r, c: torch.randn(r, c, device=DEV).to(torch.bfloat16)
a = mk(M, K); bs = [mk(K, N) for _ in range(3)]; cs = [torch.empty(M, N, device=DEV, dtype=torch.bfloat16) for _ in range(3)]
for nprob in (5, 4, 1):
    As = [mk(M, K) for _ in range(nprob)]; Bs = [mk(K, N) for _ in range(nprob)]
    c = torch.randn(M, N, device=DEV).to(torch.bfloat16); base = c.float().clone()
    descs = (_lib.GemmDesc * nprob)(*[T._fdesc(x, 0, y, 0, c, accumulate=1) for x, y in zip(As, Bs)])
    check(L := T.L.hap_matmul_batch(descs, nprob, 1, BF16, BF16, 0, 0)); torch.cuda.synchronize()
    want = base + sum(x.float() @ y.float() for x, y in zip(As, Bs))
    d = (c.float() - want).abs()
    bad = (d > 1.01 * (want.abs() * 2 ** -8 * 2 + 1e-6) + 0.6)
    idx = bad.nonzero()
    print(nprob, "rel", T.rel_err(c, want), "max abs", float(d.max()), "bad", int(bad.sum()), flush=True)
    if len(idx):
        rows = idx[:, 0].unique(); cols = idx[:, 1].unique()
        print("  rows", rows[:20].tolist(), len(rows), " cols", cols[:40].tolist(), len(cols))
        r0, c0 = idx[0].tolist(); print("  sample", r0, c0, float(c[r0, c0]), float(want[r0, c0]), float(base[r0, c0]))
