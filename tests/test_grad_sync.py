"""Gradient-synchronisation choice (host logic, CPU): the SFB rule of HAP
(PAPER.md §"Sufficient Factor Broadcasting") priced with the reference cost
model.  Few tokens per GPU make the activation factors smaller than the
weight gradient, so SFB wins; many tokens or many devices make the replicated
full-batch dW GEMM and the gathers dearer than one all-reduce."""
import pytest

import goldens
from paper_2401_05965_b200 import ClusterSpec, workloads
from paper_2401_05965_b200.executor import price_grad_sync
from paper_2401_05965_b200.program import DistributedProgram


def _choice(n, tokens_per_gpu, kdim=768, ndim=3072):
    spec = ClusterSpec.from_dict(workloads.cluster_doc(workloads.sm_caps(n)))
    return price_grad_sync(spec, None, "W", kdim, ndim, [("x", "y", tokens_per_gpu * n)])


@pytest.mark.parametrize("n,tokens,want", [(2, 256, "sfb"), (4, 256, "sfb"), (8, 256, "all_reduce"),
                                           (2, 1024, "all_reduce"), (2, 8192, "all_reduce")])
def test_sfb_rule_on_b200_clusters(n, tokens, want):
    # The MoE bench (2 sequences x 128 tokens per GPU) and the BERT bench
    # (64 x 128) sit on either side of the crossover.
    assert _choice(n, tokens) == want
    assert _choice(n, tokens, 3072, 768) == want


def test_sfb_wins_for_the_small_batch_mlp():
    # configs[0]: batch 64, hidden 1024, two devices at speed 1:2.
    spec = ClusterSpec.from_dict(goldens.load_json("clusters", "ratio12.json"))
    assert price_grad_sync(spec, (1 / 3, 2 / 3), "W1", 1024, 1024, [("x", "h", 64)]) == "sfb"


def test_sfb_price_grows_with_uses():
    # A weight used by several row-sharded matmuls gathers factors for each use.
    spec = ClusterSpec.from_dict(workloads.cluster_doc(workloads.sm_caps(2)))
    one = price_grad_sync(spec, None, "W", 768, 3072, [("x", "y", 512)])
    many = price_grad_sync(spec, None, "W", 768, 3072, [("x", "y", 512)] * 4)
    assert one == "sfb" and many == "all_reduce"


@pytest.mark.parametrize("cname", ["b200x2", "b200x4"])
def test_moe_plans_are_comm_free_forward(cname):
    # The planner shards every expert's activations by rows and replicates the
    # weights (data parallel forward); the weight gradients are then the SFB
    # candidates.
    doc = goldens.plan("moe2_b2", cname)
    prog = DistributedProgram.from_json(doc["program"])
    assert not [i for i in prog.instrs if i.is_comm]
    params = [i for i in prog.instrs if i.kind == "parameter"]
    assert len(params) == 8
