import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import test_gpu_kernels as T
from paper_2401_05965_b200 import _lib
DEV = torch.device("cuda")
M, N, K, cap = (int(v) for v in sys.argv[1:5])
mode = sys.argv[5]
a = torch.randn(M, K, device=DEV).to(torch.bfloat16)
b = (torch.randn(K, N, device=DEV) / K ** 0.5).to(torch.bfloat16)
c = torch.zeros(M, N, device=DEV, dtype=torch.bfloat16)
r = torch.randn(M, N, device=DEV).to(torch.bfloat16)
want = a.float() @ b.float()
if mode == "plain":
    T._run_descs([T._fdesc(a, 0, b, 0, c)], sm_cap=cap)
elif mode == "acc":
    c.copy_(r); T._run_descs([T._fdesc(a, 0, b, 0, c, accumulate=1)], sm_cap=cap); want = want + r.float()
elif mode == "add":
    T._run_descs([T._fdesc(a, 0, b, 0, c, epi=_lib.EPI_ADD, R=r)], sm_cap=cap); want = want + r.float()
elif mode == "add_scalar":
    rr = torch.randn(M * N + 1, device=DEV).to(torch.bfloat16)
    rv = rr[1:].view(M, N)
    d = T._fdesc(a, 0, b, 0, c, epi=_lib.EPI_ADD)
    d.R, d.ldr = rv.data_ptr(), N
    T._run_descs([d], sm_cap=cap); want = want + rv.float()
elif mode == "swish":
    y, z = torch.empty_like(c), torch.empty_like(c)
    T._run_descs([T._fdesc(a, 0, b, 0, c, epi=_lib.EPI_SWISH, epi_tag=3, Y=y, Z=z)], sm_cap=cap)
torch.cuda.synchronize()
print(mode, M, N, K, cap, "err", T.rel_err(c, want), flush=True)
