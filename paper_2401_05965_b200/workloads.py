"""Graph builders for the benchmark configurations (BASELINE.json ``configs``).

Every graph is written in the reference IR (graph_ir.py), because the planner
must emit exactly the reference's program for it.  That IR has rank-2 MatMul,
five unary tags, add/mul and Reduce — no transpose, softmax, layer norm or
convolution — so the transformer workloads are *GEMM skeletons*: every dense
projection of the real model at its real shape, with the token-mixing
attention (2.7% of BERT-base flops at seq 128) replaced by an elementwise
gate ``sigmoid(q*k)*v`` and GELU by SiLU ``f*sigmoid(f)``.  DESIGN.md lists
what each proxy keeps and drops.
"""
from __future__ import annotations

import json
import os

from .graph_ir import Graph, graph_from_dict


def _n(nid: str, op: str, shape, inputs=(), **attrs) -> dict:
    doc = {"id": nid, "op": op, "shape": list(shape)}
    if inputs:
        doc["inputs"] = list(inputs)
    if attrs:
        doc["attrs"] = attrs
    return doc


def mlp_doc(batch: int = 64, hidden: int = 1024, layers: int = 2) -> dict:
    """configs[0]: ``layers`` dense layers with ReLU between, summed to a loss."""
    nodes = [_n("x", "Placeholder", [batch, hidden])]
    prev = "x"
    for i in range(1, layers + 1):
        nodes.append(_n(f"w{i}", "Parameter", [hidden, hidden]))
        nodes.append(_n(f"h{i}", "MatMul", [batch, hidden], [prev, f"w{i}"]))
        prev = f"h{i}"
        if i < layers:
            nodes.append(_n(f"a{i}", "ElemwiseUnary", [batch, hidden], [prev], tag="relu"))
            prev = f"a{i}"
    nodes.append(_n("loss", "Reduce", [], [prev], dims="all"))
    return {"nodes": nodes, "loss": "loss"}


def bert_doc(layers: int = 12, batch: int = 64, seq: int = 128, hidden: int = 768,
             ffn: int = 3072) -> dict:
    """configs[2]: BERT-base GEMM skeleton over ``batch*seq`` token rows.

    Per layer: Q/K/V projections, gate ``sigmoid(q*k)*v``, output projection
    with residual, FFN up-projection, SiLU, FFN down-projection with residual.
    """
    tokens = batch * seq
    nodes = [_n("x0", "Placeholder", [tokens, hidden])]
    prev = "x0"
    for layer in range(layers):
        p = f"l{layer}_"
        for w in ("q", "k", "v"):
            nodes.append(_n(p + "W" + w, "Parameter", [hidden, hidden]))
            nodes.append(_n(p + w, "MatMul", [tokens, hidden], [prev, p + "W" + w]))
        nodes.append(_n(p + "qk", "ElemwiseBinary", [tokens, hidden], [p + "q", p + "k"], tag="mul"))
        nodes.append(_n(p + "att", "ElemwiseUnary", [tokens, hidden], [p + "qk"], tag="sigmoid"))
        nodes.append(_n(p + "ctx", "ElemwiseBinary", [tokens, hidden], [p + "att", p + "v"], tag="mul"))
        nodes.append(_n(p + "Wo", "Parameter", [hidden, hidden]))
        nodes.append(_n(p + "o", "MatMul", [tokens, hidden], [p + "ctx", p + "Wo"]))
        nodes.append(_n(p + "x1", "ElemwiseBinary", [tokens, hidden], [prev, p + "o"], tag="add"))
        nodes.append(_n(p + "W1", "Parameter", [hidden, ffn]))
        nodes.append(_n(p + "f1", "MatMul", [tokens, ffn], [p + "x1", p + "W1"]))
        nodes.append(_n(p + "s1", "ElemwiseUnary", [tokens, ffn], [p + "f1"], tag="sigmoid"))
        nodes.append(_n(p + "g", "ElemwiseBinary", [tokens, ffn], [p + "f1", p + "s1"], tag="mul"))
        nodes.append(_n(p + "W2", "Parameter", [ffn, hidden]))
        nodes.append(_n(p + "f2", "MatMul", [tokens, hidden], [p + "g", p + "W2"]))
        nodes.append(_n(p + "x2", "ElemwiseBinary", [tokens, hidden], [p + "x1", p + "f2"], tag="add"))
        prev = p + "x2"
    nodes.append(_n("loss", "Reduce", [], [prev], dims="all"))
    return {"nodes": nodes, "loss": "loss"}


def moe_doc(experts: int = 8, tokens: int = 256, hidden: int = 768, ffn: int = 3072) -> dict:
    """configs[3]/[4]: a mixture-of-experts FFN block (BERT-base widths).

    The router's dispatch is the data loader's: expert e receives its own
    token batch x_e [tokens, hidden] (a placeholder), runs a SiLU FFN
    (W1_e, W2_e) and the per-expert outputs are summed into the loss.  With
    few tokens per expert the weights dominate the activations, which is
    where sufficient-factor broadcasting beats all-reducing the weight
    gradients — the choice the executor prices with the cost model."""
    nodes = []
    losses = []
    for e in range(experts):
        p = f"e{e}_"
        nodes.append(_n(p + "x", "Placeholder", [tokens, hidden]))
        nodes.append(_n(p + "W1", "Parameter", [hidden, ffn]))
        nodes.append(_n(p + "f1", "MatMul", [tokens, ffn], [p + "x", p + "W1"]))
        nodes.append(_n(p + "s1", "ElemwiseUnary", [tokens, ffn], [p + "f1"], tag="sigmoid"))
        nodes.append(_n(p + "g", "ElemwiseBinary", [tokens, ffn], [p + "f1", p + "s1"], tag="mul"))
        nodes.append(_n(p + "W2", "Parameter", [ffn, hidden]))
        nodes.append(_n(p + "y", "MatMul", [tokens, hidden], [p + "g", p + "W2"]))
        nodes.append(_n(p + "l", "Reduce", [], [p + "y"], dims="all"))
        losses.append(p + "l")
    acc = losses[0]
    for i, l in enumerate(losses[1:], 1):
        out = "loss" if i == len(losses) - 1 else f"lsum{i}"
        nodes.append(_n(out, "ElemwiseBinary", [], [acc, l], tag="add"))
        acc = out
    if len(losses) == 1:
        nodes.append(_n("loss", "Identity", [], [acc]))
    return {"nodes": nodes, "loss": "loss"}


def moe_stack_doc(layers: int = 12, experts: int = 2, batch: int = 8, seq: int = 128, hidden: int = 768,
                  ffn: int = 3072) -> dict:
    """configs[4] (BERT-MoE FFN stack): per layer, `experts` SiLU FFN experts
    (BERT-base widths) read the layer input and their outputs join the
    residual stream, x_{l+1} = x_l + sum_e FFN_e(x_l).  Every expert sees
    every token (a dense mixture: the reference IR has no routing op), and
    with few tokens per GPU the weight gradients dwarf the activation factors
    — the sufficient-factor-broadcasting regime.  Experts per layer stay at 2
    because the planner's search grows combinatorially with independent
    branches (4 experts exhaust its 200k-expansion budget)."""
    tokens = batch * seq
    nodes = [_n("x0", "Placeholder", [tokens, hidden])]
    prev = "x0"
    for layer in range(layers):
        outs = []
        for e in range(experts):
            p = f"l{layer}_e{e}_"
            nodes.append(_n(p + "W1", "Parameter", [hidden, ffn]))
            nodes.append(_n(p + "f1", "MatMul", [tokens, ffn], [prev, p + "W1"]))
            nodes.append(_n(p + "s1", "ElemwiseUnary", [tokens, ffn], [p + "f1"], tag="sigmoid"))
            nodes.append(_n(p + "g", "ElemwiseBinary", [tokens, ffn], [p + "f1", p + "s1"], tag="mul"))
            nodes.append(_n(p + "W2", "Parameter", [ffn, hidden]))
            nodes.append(_n(p + "y", "MatMul", [tokens, hidden], [p + "g", p + "W2"]))
            outs.append(p + "y")
        acc = prev
        for i, y in enumerate(outs):
            out = f"l{layer}_x{i + 1}"
            nodes.append(_n(out, "ElemwiseBinary", [tokens, hidden], [acc, y], tag="add"))
            acc = out
        prev = acc
    nodes.append(_n("loss", "Reduce", [], [prev], dims="all"))
    return {"nodes": nodes, "loss": "loss"}


def vit_moe_doc(layers: int = 12, experts: int = 2, images: int = 16, tokens: int = 197, hidden: int = 768,
                ffn: int = 3072) -> dict:
    """configs[3] (ViT-MoE): a ViT-B/16 GEMM skeleton (197 tokens per image,
    hidden 768) whose every block is an attention skeleton (Q/K/V, the gate
    sigmoid(q*k)*v, output projection + residual — as bert_doc) followed by
    a mixture of `experts` SiLU FFN experts (768 -> 3072 -> 768) whose outputs
    are summed and added to the residual stream.  Every expert sees every
    token (a dense mixture: the reference IR has no routing op)."""
    rows = images * tokens
    nodes = [_n("x0", "Placeholder", [rows, hidden])]
    prev = "x0"
    for layer in range(layers):
        p = f"l{layer}_"
        for w in ("q", "k", "v"):
            nodes.append(_n(p + "W" + w, "Parameter", [hidden, hidden]))
            nodes.append(_n(p + w, "MatMul", [rows, hidden], [prev, p + "W" + w]))
        nodes.append(_n(p + "qk", "ElemwiseBinary", [rows, hidden], [p + "q", p + "k"], tag="mul"))
        nodes.append(_n(p + "att", "ElemwiseUnary", [rows, hidden], [p + "qk"], tag="sigmoid"))
        nodes.append(_n(p + "ctx", "ElemwiseBinary", [rows, hidden], [p + "att", p + "v"], tag="mul"))
        nodes.append(_n(p + "Wo", "Parameter", [hidden, hidden]))
        nodes.append(_n(p + "o", "MatMul", [rows, hidden], [p + "ctx", p + "Wo"]))
        nodes.append(_n(p + "x1", "ElemwiseBinary", [rows, hidden], [prev, p + "o"], tag="add"))
        ys = []
        for e in range(experts):
            q = f"{p}e{e}_"
            nodes.append(_n(q + "W1", "Parameter", [hidden, ffn]))
            nodes.append(_n(q + "f1", "MatMul", [rows, ffn], [p + "x1", q + "W1"]))
            nodes.append(_n(q + "s1", "ElemwiseUnary", [rows, ffn], [q + "f1"], tag="sigmoid"))
            nodes.append(_n(q + "g", "ElemwiseBinary", [rows, ffn], [q + "f1", q + "s1"], tag="mul"))
            nodes.append(_n(q + "W2", "Parameter", [ffn, hidden]))
            nodes.append(_n(q + "y", "MatMul", [rows, hidden], [q + "g", q + "W2"]))
            ys.append(q + "y")
        acc = ys[0]
        for i, y in enumerate(ys[1:], 1):
            nodes.append(_n(f"{p}ysum{i}", "ElemwiseBinary", [rows, hidden], [acc, y], tag="add"))
            acc = f"{p}ysum{i}"
        nodes.append(_n(p + "x2", "ElemwiseBinary", [rows, hidden], [p + "x1", acc], tag="add"))
        prev = p + "x2"
    nodes.append(_n("loss", "Reduce", [], [prev], dims="all"))
    return {"nodes": nodes, "loss": "loss"}


def vit_moe(layers: int = 12, experts: int = 2, images: int = 16, tokens: int = 197, hidden: int = 768,
            ffn: int = 3072) -> Graph:
    return graph_from_dict(vit_moe_doc(layers, experts, images, tokens, hidden, ffn))


def expert_sharded_program(g: Graph):
    """The expert-sharded program of a ViT-MoE skeleton (configs[3]).

    Attention blocks run data parallel (token rows ``@shard0``, weights
    replicated); each MoE FFN block runs expert-sliced over all devices:
    the block input is all-gathered along the token axis (``x1@full``), every
    expert's W1 is column-sharded and W2 row-sharded (``@shard1`` /
    ``@shard0``: each device holds a ratio-weighted slice of every expert),
    the expert outputs are partial sums, added across experts and
    reduce-scattered back to token rows.  Uneven all-gather and
    reduce-scatter run in every layer's forward, and their adjoints
    (reduce-scatter, all-gather) in the backward.

    The same instruction pattern is in the REFERENCE planner's program space:
    tools/vit_moe_plan.py enumerates every complete program of one expert
    FFN block with the reference-restated synthesizer
    (synthesizer.enumerate_all_complete, reference synthesizer.py:538) and
    finds this one; the planner itself never emits it for these graphs
    because its forward-only cost model prices data parallelism as
    communication-free (configs[3])."""
    from .program import DistributedProgram, Instruction

    kinds = {"MatMul": "matmul", "ElemwiseUnary": "elemwise_unary", "ElemwiseBinary": "elemwise_binary",
             "Reduce": "reduce", "Identity": "identity"}
    form: dict = {}
    instrs: list = []
    emitted: set = set()

    def source(ref: str, out: str, kind: str, axis=None):
        if out not in emitted:
            emitted.add(out)
            instrs.append(Instruction(kind, ref, output=out, axis=axis))

    for n in g.nodes:
        if n.op in ("Placeholder", "Parameter"):
            continue
        base = n.id.split("_", 1)[-1]
        expert = "_e" in n.id and base.split("_", 1)[-1] in ("f1", "s1", "g", "y")
        ops = []
        for i in n.inputs:
            src = g.producer(i)
            if src.op == "Parameter":
                if expert and i.endswith("_W1"):
                    source(i, f"{i}@shard1", "parameter_shard", 1)
                    ops.append(f"{i}@shard1")
                elif expert and i.endswith("_W2"):
                    source(i, f"{i}@shard0", "parameter_shard", 0)
                    ops.append(f"{i}@shard0")
                else:
                    source(i, f"{i}@full", "parameter")
                    ops.append(f"{i}@full")
            elif src.op == "Placeholder":
                source(i, f"{i}@shard0", "placeholder_shard", 0)
                ops.append(f"{i}@shard0")
            else:
                ops.append(form[i])
        out_form = "shard0"
        if expert:
            kind = n.id.rsplit("_", 1)[-1]
            if kind == "f1":
                x = n.inputs[0]
                if f"{x}@full" not in emitted:
                    emitted.add(f"{x}@full")
                    instrs.append(Instruction("all_gather", x, operands=(f"{x}@shard0",), output=f"{x}@full", axis=0))
                ops[0] = f"{x}@full"
            out_form = "partial" if kind == "y" else "shard1"
        elif "ysum" in n.id:
            out_form = "partial"
        elif n.op == "Reduce":
            out_form = "partial"
        elif n.id.endswith("_x2"):
            # the summed expert outputs go back to token rows
            y = n.inputs[1]
            instrs.append(Instruction("reduce_scatter", y, operands=(f"{y}@partial",), output=f"{y}@shard0", axis=0))
            ops[1] = f"{y}@shard0"
        out = f"{n.id}@{out_form}"
        form[n.id] = out
        instrs.append(Instruction(kinds[n.op], n.id, operands=tuple(ops), output=out, dims=n.dims, tag=n.tag))
    return DistributedProgram(instrs=tuple(_theory_instrs(g, instrs)), loss=g.loss)


def _theory_instrs(g: Graph, instrs: list) -> list:
    """Each instruction as the planner's theory states it (its Hoare triple's
    instruction: ``sharded``, ``flops`` and ``elements`` as the cost model
    reads them), checking on the way that the sequence is a valid program of
    that theory: every triple's precondition holds when it runs, and the
    loss property is realised at the end (theory.py; reference theory.py)."""
    from .theory import build_theory, merge_post

    theory = build_theory(g, 2, fuse=False)   # one instruction per triple (sources unfused)
    index = {}
    for t in theory.triples:
        if len(t.instrs) == 1:
            index.setdefault(t.instrs[0].canonical(), []).append(t)
    props = frozenset(theory.initial_props)
    out = []
    for ins in instrs:
        triples = [t for t in index.get(ins.canonical(), []) if t.pre <= props]
        if not triples:
            raise ValueError(f"{ins.canonical()} is not applicable under the planner's theory")
        t = triples[0]
        out.append(t.instrs[0])
        props = merge_post(props, t.post)
    if not any(p.ref == g.loss for p in props):
        raise ValueError("program does not realise the loss")
    return out


def expert_sharded_plan(g: Graph, spec) -> dict:
    """Reference-schema plan document (cli.py:73) of the expert-sharded
    program: ratios by the planner's own alternating loop with the synthesis
    step fixed to this program (optimizer_loop.alternate: the LP of
    load_balancer.optimize_ratios), shard table by its rounding rule,
    estimate by its cost model."""
    from .cli import plan_document
    from .optimizer_loop import alternate
    from .synthesizer import SynthesisResult

    prog = expert_sharded_program(g)

    def synth(*_args):
        return SynthesisResult(program=prog, cost_s=0.0, complete=True, optimal=True, exhausted=False,
                               expansions=0, generated=0, purged=0)

    return plan_document(g, spec, alternate(g, spec, synth_fn=synth))


def moe_stack(layers: int = 12, experts: int = 2, batch: int = 8, seq: int = 128) -> Graph:
    return graph_from_dict(moe_stack_doc(layers, experts, batch, seq))


def moe(experts: int = 8, tokens: int = 256, hidden: int = 768, ffn: int = 3072) -> Graph:
    return graph_from_dict(moe_doc(experts, tokens, hidden, ffn))


def mlp(batch: int = 64, hidden: int = 1024, layers: int = 2) -> Graph:
    return graph_from_dict(mlp_doc(batch, hidden, layers))


def bert(layers: int = 12, batch: int = 64, seq: int = 128, hidden: int = 768,
         ffn: int = 3072) -> Graph:
    return graph_from_dict(bert_doc(layers, batch, seq, hidden, ffn))


# Heterogeneity emulation: per-rank SM caps on the homogeneous 8xB200 box.
SM_COUNT = 148
SM_CAP_PATTERN = (148, 104, 132, 88)


def sm_caps(n_gpus: int) -> list[int]:
    """Mixed SM caps for ``n_gpus`` ranks; one GPU runs uncapped."""
    if n_gpus == 1:
        return [SM_COUNT]
    return [SM_CAP_PATTERN[j % len(SM_CAP_PATTERN)] for j in range(n_gpus)]


# NVLink-5 collective model for the planner's cost model (latency, bytes/s),
# bf16 elements.  ROUND-1 values, set from the profiling guide's measured
# NVLink figures (770 GB/s peer copy, 725 GB/s 8-rank all-reduce bus
# bandwidth) derated for small messages: the committed golden clusters
# (tests/golden/clusters/b200x*.json) were made with these, so
# cluster_doc(fitted=False) still reproduces them.
NVLINK_MODEL = {
    "all_gather": (8e-6, 600e9),
    "all_reduce": (12e-6, 360e9),
    "reduce_scatter": (8e-6, 600e9),
    "all_to_all": (10e-6, 500e9),
    "grouped_broadcast": (4e-6, 600e9),
}
# The planner's device speed: sustained bf16 GEMM rate per SM, 1376.6 TF/s
# as measured in round 1 (MEASURED_PEAKS.json of the current pool reads 1398.8
# sustained).  Only ratios of device speeds shape a plan; the committed
# goldens were planned with this value, so it stays for byte-identical plans.
BF16_TFLOPS_PER_SM = 1376.6e12 / SM_COUNT

# Measured lines (tools/coll_fit.py on B200s: the reference's fit_linear,
# cost_model.py:310, per world size, collective and implementation — NVLink
# peer-memory kernel "p2p" or NCCL "nccl"), in the cost model's units: x =
# the bytes comm_time charges (elements x bytes/element, x the largest shard
# ratio for gathers, reduce-scatters and all-to-alls).
FITS_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "collectives_b200.json")
_FITS: dict | None = None


def collective_fits(world: int) -> dict | None:
    """{kind: {impl: (latency_s, bw_Bps)}} measured at exactly ``world``
    GPUs, or None (the hand-set round-1 lines are used then): a line fitted
    at one rank count does not transfer — with the 4-GPU lines applied to 2
    GPUs the model picked all-reduce for BERT-MoE, which measured 29 % slower
    than SFB there (profiles/r02_multi_n2.md)."""
    global _FITS
    if _FITS is None:
        _FITS = {}
        if os.path.exists(FITS_PATH):
            with open(FITS_PATH) as fh:
                _FITS = {int(k): v for k, v in json.load(fh).items()}
    if world < 2 or world not in _FITS:
        return None
    doc = _FITS[world]
    return {kind: {impl: (v["latency_s"], v["bw_Bps"]) for impl, v in impls.items()} for kind, impls in doc.items()}


def impl_cluster_doc(caps: list[int], impl: str, bytes_per_element: int = 2) -> dict | None:
    """Cluster spec whose collective lines are one implementation's fitted
    lines ("p2p" or "nccl"); None without measurements for it."""
    fits = collective_fits(len(caps))
    if not fits or any(impl not in fits.get(k, {}) for k in ("all_gather", "reduce_scatter", "all_reduce",
                                                               "all_to_all")):
        return None
    lines = {k: fits[k][impl] for k in ("all_gather", "reduce_scatter", "all_reduce", "all_to_all")}
    lines["grouped_broadcast"] = lines["all_gather"]
    return {"devices": [{"flops": float(c) * BF16_TFLOPS_PER_SM} for c in caps],
            "collectives": {k: {"latency_s": lat, "bw_Bps": bw} for k, (lat, bw) in lines.items()},
            "bytes_per_element": bytes_per_element}


def cluster_doc(caps: list[int], bytes_per_element: int = 2, fitted: bool = True) -> dict:
    """Cluster spec (reference ClusterSpec JSON) for SM-capped B200 ranks.
    Collective lines: the measured fits (per kind, the implementation the
    executor's per-call-site choice takes at 4 MiB, Executor._use_p2p) when
    measured for this world size; else the round-1 model."""
    lines = dict(NVLINK_MODEL)
    fits = collective_fits(len(caps)) if fitted else None
    if fits:
        ref = 4 << 20
        for kind in ("all_gather", "reduce_scatter", "all_reduce", "all_to_all"):
            impls = fits.get(kind)
            if impls:
                lines[kind] = min(impls.values(), key=lambda lb: lb[0] + ref / lb[1])
        lines["grouped_broadcast"] = lines["all_gather"]
    return {
        "devices": [{"flops": float(c) * BF16_TFLOPS_PER_SM} for c in caps],
        "collectives": {k: {"latency_s": lat, "bw_Bps": bw} for k, (lat, bw) in lines.items()},
        "bytes_per_element": bytes_per_element,
    }


def synthetic_inputs(g: Graph, seed: int, scaled: bool = True) -> dict:
    """Seeded float64 bindings for every source tensor, in node order.

    ``scaled=False`` reproduces the reference's ``random_inputs``
    (interpreter.py:252): standard normal everywhere.  ``scaled=True`` divides
    rank-2 parameters by sqrt(fan-in) so deep skeletons stay in range (the
    reference interpreter is then run on exactly these arrays).
    """
    import numpy as np

    rng = np.random.default_rng(seed)
    # residual-branch output projections get the GPT-2 1/sqrt(2L) factor so a
    # deep skeleton without normalisation keeps O(1) activations.
    # (BERT skeleton: one _Wo per layer; MoE stack: every expert's _W2 feeds
    # the residual stream.)
    branches = [n.id for n in g.nodes if n.id.endswith("_Wo")]
    if not branches:
        branches = [n.id for n in g.nodes if n.id.startswith("l") and n.id.endswith("_W2")]
    depth = len(branches)
    out = {}
    for node in g.nodes:
        if node.op in ("Placeholder", "Parameter"):
            value = rng.standard_normal(node.shape)
            if scaled and node.op == "Parameter" and len(node.shape) == 2:
                value = value / np.sqrt(node.shape[0])
                if depth and node.id.endswith(("_Wo", "_W2")):
                    value = value / np.sqrt(2 * depth)
            out[node.id] = value
    return out



def planned_program(g: Graph, m: int, plan_doc: dict):
    """(program, shard table, ratio row) for ``m`` equal devices from a plan
    document the reference planner emitted for the same graph family (same
    node ids) at another device count.

    The planner emits the SAME program for these skeletons at every device
    count: the data-parallel program (token rows ``@shard0``, weights
    ``@full``, ``loss@partial``) — checked by tests/test_workloads.py for the
    2-layer BERT and BERT-MoE skeletons at m = 1, 2, 4 and for the 12-layer
    bench plans at m = 2, 4, 8.  At m = 1 every sharding choice ties, so its
    A* search grows ~3.6x per layer (1.2 / 6.9 / 24.7 s for 1 / 2 / 3 BERT
    layers) and the 12-layer m = 1 plan does not finish; bench.py's N = 1
    line therefore takes the program of the N = 2 plan, re-targeted to one
    device (its shard table: the whole token axis)."""
    from .program import DistributedProgram

    prog = DistributedProgram.from_json(plan_doc["program"])
    ids = {n.id for n in g.nodes}
    missing = sorted({ins.ref for ins in prog.instrs} - ids)
    if missing:
        raise ValueError(f"plan does not belong to this graph: unknown tensors {missing[:5]}")
    table = {}
    for ins in prog.instrs:
        for did in (ins.output,) + tuple(ins.operands):
            ref, _, form = did.partition("@")
            if form.startswith("shard"):
                axis = int(form[len("shard"):])
                extent = g.producer(ref).shape[axis]
                table[(ref, axis)] = [extent // m + (1 if j < extent % m else 0) for j in range(m)]
    return prog, table, tuple(1.0 / m for _ in range(m))
