import sys, torch
sys.path.insert(0, ".")
from paper_2401_05965_b200 import _lib
from paper_2401_05965_b200._lib import BF16, F32, check
L = _lib.lib()
dev = torch.device("cuda")
def run(M, N, K, ta, tb, out, acc=0):
    a = torch.randn((K, M) if ta else (M, K), device=dev).to(torch.bfloat16)
    b = torch.randn((N, K) if tb else (K, N), device=dev).to(torch.bfloat16)
    c = torch.randn((M, N), device=dev).to(out)
    base = c.float().clone()
    eng = L.hap_matmul_engine(a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb, M, N, K, BF16)
    check(L.hap_matmul(a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb, c.data_ptr(), N, M, N, K, BF16,
                       BF16 if out == torch.bfloat16 else F32, acc, 0, 0))
    torch.cuda.synchronize()
    want = (a.float().t() if ta else a.float()) @ (b.float().t() if tb else b.float()) + (base if acc else 0)
    err = ((c.float() - want).abs().max() / want.abs().max()).item()
    bad = ((c.float() - want).abs() > 0.05 * want.abs().max()).nonzero()
    print(f"M={M} N={N} K={K} ta={ta} tb={tb} out={out} acc={acc} eng={eng} err={err:.2e} bad={bad.shape[0]} first={bad[:3].tolist()}")
for (M, N, K) in [(21, 1024, 1024), (1024, 1024, 21), (11, 32, 32), (32, 32, 11), (5, 32, 32), (32, 32, 5), (43, 1024, 1024), (1024, 1024, 43), (16, 32, 32), (32, 32, 16)]:
    for ta, tb in [(0, 0), (0, 1), (1, 0), (1, 1)]:
        for out in (torch.bfloat16, torch.float32):
            run(M, N, K, ta, tb, out)
run(32, 32, 11, 1, 0, torch.float32, acc=1)
