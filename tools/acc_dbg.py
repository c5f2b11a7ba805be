import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import test_gpu_kernels as T
from paper_2401_05965_b200 import _lib
DEV = torch.device("cuda")
torch.manual_seed(11)
M, N, K = 1024, 768, 512
mk = lambda r, c: torch.randn(r, c, device=DEV).to(torch.bfloat16)
for nprob in (1, 2, 4, 5):
    As = [mk(M, K) for _ in range(nprob)]; Bs = [mk(K, N) for _ in range(nprob)]
    c = torch.randn(M, N, device=DEV).to(torch.bfloat16); base = c.float().clone()
    descs = [T._fdesc(x, 0, y, 0, c, accumulate=1) for x, y in zip(As, Bs)]
    T._run_descs(descs, sum_k=1)
    want = base + sum(x.float() @ y.float() for x, y in zip(As, Bs))
    d = (c.float() - want).abs()
    ulp = want.abs().clamp_min(1e-3) * 2 ** -8
    print(nprob, "max abs", float(d.max()), "max ulps", float((d / ulp).max()), "rel", T.rel_err(c, want), flush=True)
