import sys, json, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import goldens
from oracle import interpreter_np as O
from paper_2401_05965_b200.executor import ExecConfig, Executor, LocalGroup
from paper_2401_05965_b200.program import DistributedProgram
from paper_2401_05965_b200.sharding import table_from_plan
from paper_2401_05965_b200 import _lib
gname, cname, dtype = "chain4", "hetero2", "bf16"
g = goldens.graph(gname); doc = goldens.plan(gname, cname); vals = goldens.values(gname, cname)
inputs = goldens.inputs(g, vals, 0)
prog = DistributedProgram.from_json(doc["program"]); m = doc["devices"]
shapes = {n.id: n.shape for n in g.sources()}
ex = Executor(prog, m, table_from_plan(doc), shapes, group=LocalGroup(m), config=ExecConfig(dtype=dtype, input_grads=True))
ex.load(inputs); ex.forward(); ex.backward(); ex.stream.synchronize()
h4 = ex.tensor("h4@shard0", 1).float(); u4 = ex.tensor("u4@shard0", 1).float()
gu4 = ex.grads[("u4@shard0", 1)]; gh4 = ex.grads[("h4@shard0", 1)]
print("h4", h4[0,:8]); print("u4", u4[0,:8])
print("du4", gu4.tensor[:8].float()); print("dh4", gh4.tensor[:8].float())
print("ptrs", gu4.ptr, gh4.ptr, ex.bufs[("h4@shard0",1)].ptr, ex.bufs[("u4@shard0",1)].ptr)
for op in ex.ops_bwd:
    if op.what in ("hap_unary_grad",):
        print(op.what, op.args[:11])
# direct kernel call
L = _lib.lib()
out = torch.zeros(160, dtype=torch.bfloat16, device="cuda")
x = ex.bufs[("h4@shard0",1)]; y = ex.bufs[("u4@shard0",1)]
st = L.hap_unary_grad(2, x.ptr, y.ptr, 1, gu4.ptr, 1, out.data_ptr(), 1, 160, 0, 0, 0); torch.cuda.synchronize()
print("direct", st, out[:8].float())
