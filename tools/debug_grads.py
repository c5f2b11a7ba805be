import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import goldens
from oracle import interpreter_np as O
from test_gpu_executor import _run, rounded
for gname, cname in [("chain4", "hetero2"), ("chain4", "homog2"), ("mlp", "ratio12"), ("bert2_b2", "b200x2"), ("matmul_unary", "hetero2")]:
    g = goldens.graph(gname); doc = goldens.plan(gname, cname); vals = goldens.values(gname, cname)
    inputs = goldens.inputs(g, vals, 0)
    for dtype in ("bf16", "fp32"):
        ex = _run(doc, g, inputs, dtype)
        want = O.grad_single(g, rounded(inputs, dtype))
        for ref, value in want.items():
            for r, forms in ex.gradient(ref).items():
                for did, grad in forms:
                    grad = grad.float().cpu().numpy().astype(np.float64)
                    if "@shard" in did:
                        axis = int(did.rsplit("shard", 1)[1]); sizes = ex._sizes(ref, axis); off = int(np.sum(sizes[:r]))
                        exp = np.take(value, np.arange(off, off + sizes[r]), axis=axis)
                    else:
                        exp = value
                    if not exp.size: continue
                    mx = np.max(np.abs(grad - exp)) / np.max(np.abs(exp))
                    fro = np.linalg.norm(grad - exp) / np.linalg.norm(exp)
                    frac = np.mean(np.abs(grad - exp) > 2e-2 * np.max(np.abs(exp)))
                    print(f"{gname}.{cname} {dtype} {did} r{r}: max {mx:.2e} fro {fro:.2e} outliers {frac:.2%}")
