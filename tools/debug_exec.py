import sys, json, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import goldens
from oracle import interpreter_np as O
from paper_2401_05965_b200.executor import ExecConfig, Executor, LocalGroup
from paper_2401_05965_b200.program import DistributedProgram
from paper_2401_05965_b200.sharding import table_from_plan
gname, cname, dtype = sys.argv[1], sys.argv[2], sys.argv[3]
g = goldens.graph(gname); doc = goldens.plan(gname, cname); vals = goldens.values(gname, cname)
inputs = goldens.inputs(g, vals, goldens.seeds(vals)[0])
prog = DistributedProgram.from_json(doc["program"]); m = doc["devices"]
shapes = {n.id: n.shape for n in g.sources()}
ex = Executor(prog, m, table_from_plan(doc), shapes, group=LocalGroup(m), config=ExecConfig(dtype=dtype, input_grads=True))
ex.load(inputs); ex.forward(); ex.stream.synchronize()
program, m2, table = O.load_plan(doc)
env, losses = O.run_distributed(program, m2, inputs, table)
for did in env:
    for r in range(m):
        got = ex.tensor(did, r).float().cpu().numpy(); want = env[did][r]
        e = np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-6) if want.size else 0
        if e > 1e-2: print("FWD", did, r, got.shape, e)
ex.backward(); ex.stream.synchronize()
grads = O.backward_distributed(program, m2, env, table)
for (did, r), gb in sorted(ex.grads.items()):
    got = gb.tensor[:gb.numel].view(gb.shape).float().cpu().numpy(); want = grads[did][r]
    e = np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-6) if want.size else 0
    print("BWD", did, r, gb.shape, "dtype", gb.dtype, f"{e:.3e}")
for op in ex.ops_bwd[:40]:
    print(op.what, [a for a in op.args if not isinstance(a, int) or a < 1<<20][:12])
