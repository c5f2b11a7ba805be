"""Hoare-triple background theory of a graph (reference theory.py).

DERIVED FROM THE REFERENCE: this module restates shardplan/theory.py closely —
north_star requires the planner to emit exactly the reference's programs,
ratios and estimates, and the goldens check it byte for byte — so it is not
original work of this repository; the executor, the kernels and the
collectives are.

A triple ``{pre} instrs {post}`` says: if the partial program realises every
property in ``pre``, appending ``instrs`` realises ``post``.  Properties are
``e|Id``, ``e|AG(d)``, ``e|AR`` (program.py) plus two search guards
(``Comm`` / ``NotComm``).  The search indexes triples by position and breaks
ties on that index, so the derivation order below is part of the contract:
per node in graph order its operator rules, then per node its collective
rules, then the optional guard and fusion rewrites.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

from .graph_ir import Graph, Node, node_flops
from .program import (ALL_GATHER, ALL_REDUCE, COMM_KINDS, COMMUNICATED, GUARD_KINDS, IDENTITY,
                      NOT_COMMUNICATED, SOURCE_KINDS, Instruction, Property, all_gather, all_reduce,
                      communicated, dist_id, form_of_dist_id, identity, not_communicated)

__all__ = ["HoareTriple", "Theory", "derive_theory", "fuse_empty_preconditions",
           "add_communication_guards", "build_theory", "merge_post", "theory_to_json",
           "Instruction", "Property", "dist_id", "form_of_dist_id", "identity", "all_gather",
           "all_reduce", "communicated", "not_communicated", "IDENTITY", "ALL_GATHER",
           "ALL_REDUCE", "COMMUNICATED", "NOT_COMMUNICATED", "GUARD_KINDS", "COMM_KINDS",
           "SOURCE_KINDS"]


@dataclass(frozen=True)
class HoareTriple:
    pre: frozenset
    instrs: tuple
    post: frozenset

    def __str__(self) -> str:
        pre = ",".join(sorted(map(str, self.pre)))
        post = ",".join(sorted(map(str, self.post)))
        return "{%s} %s {%s}" % (pre, ";".join(i.canonical() for i in self.instrs), post)


@dataclass(frozen=True)
class Theory:
    triples: tuple
    loss: str
    tensor_ids: tuple
    source_ids: frozenset
    shapes: dict
    initial_props: frozenset = frozenset()


def merge_post(props: frozenset, post: frozenset) -> frozenset:
    """props ∪ post, where gaining Comm(e) drops NotComm(e)."""
    dropped = {not_communicated(p.ref) for p in post if p.kind == COMMUNICATED}
    merged = props | post
    return merged - dropped if dropped else merged


def _triple(pre, instr: Instruction, post) -> HoareTriple:
    return HoareTriple(frozenset(pre), (instr,), frozenset(post))


def _size(shape) -> int:
    out = 1
    for e in shape:
        out *= e
    return out


# --------------------------------------------------------------------- operator rules

def _sources(node: Node) -> list:
    kind = "placeholder" if node.op == "Placeholder" else "parameter"
    e = node.id
    rules = [_triple((), Instruction(kind, e, output=dist_id(e, identity(e))), {identity(e)})]
    for d in range(len(node.shape)):
        p = all_gather(e, d)
        rules.append(_triple((), Instruction(kind + "_shard", e, axis=d, output=dist_id(e, p),
                                             sharded=True), {p}))
    return rules


def _matmul(node: Node, g: Graph) -> list:
    lhs, rhs = node.inputs
    out = node.id
    work = node_flops(g, node)
    # (lhs form, rhs form, out form, sharded): row-split, column-split,
    # contraction-split (partial sums), full replication.
    forms = [(all_gather(lhs, 0), identity(rhs), all_gather(out, 0), True),
             (identity(lhs), all_gather(rhs, 1), all_gather(out, 1), True),
             (all_gather(lhs, 1), all_gather(rhs, 0), all_reduce(out), True),
             (identity(lhs), identity(rhs), identity(out), False)]
    return [_triple((a, b), Instruction("matmul", out, operands=(dist_id(lhs, a), dist_id(rhs, b)),
                                        output=dist_id(out, c), sharded=sh, flops=work), {c})
            for a, b, c, sh in forms]


def _unary(node: Node, g: Graph) -> list:
    (src,) = node.inputs
    out = node.id
    work = node_flops(g, node)
    kind = "identity" if node.op == "Identity" else "elemwise_unary"

    def mk(p_in, p_out, sh):
        return _triple((p_in,), Instruction(kind, out, operands=(dist_id(src, p_in),),
                                            output=dist_id(out, p_out), tag=node.tag, sharded=sh,
                                            flops=work), {p_out})

    rules = [mk(all_gather(src, d), all_gather(out, d), True) for d in range(len(node.shape))]
    rules.append(mk(identity(src), identity(out), False))
    if node.op == "Identity":  # linear: commutes with the cross-device sum
        rules.append(mk(all_reduce(src), all_reduce(out), False))
    return rules


def _binary(node: Node, g: Graph) -> list:
    lhs, rhs = node.inputs
    out = node.id
    work = node_flops(g, node)

    def mk(pa, pb, pc, sh):
        return _triple((pa, pb), Instruction("elemwise_binary", out,
                                             operands=(dist_id(lhs, pa), dist_id(rhs, pb)),
                                             output=dist_id(out, pc), tag=node.tag, sharded=sh,
                                             flops=work), {pc})

    rules = [mk(all_gather(lhs, d), all_gather(rhs, d), all_gather(out, d), True)
             for d in range(len(node.shape))]
    rules.append(mk(identity(lhs), identity(rhs), identity(out), False))
    if node.tag == "add":  # sums of partials add; products do not
        rules.append(mk(all_reduce(lhs), all_reduce(rhs), all_reduce(out), False))
    return rules


def _reduce(node: Node, g: Graph) -> list:
    (src,) = node.inputs
    out = node.id
    work = node_flops(g, node)
    dims = node.dims or ()

    def mk(p_in, p_out, sh):
        return _triple((p_in,), Instruction("reduce", out, operands=(dist_id(src, p_in),),
                                            output=dist_id(out, p_out), dims=dims, sharded=sh,
                                            flops=work), {p_out})

    rules = [mk(identity(src), identity(out), False), mk(all_reduce(src), all_reduce(out), False)]
    for d in range(len(g.tensors[src].shape)):
        if d in dims:
            # summing over the split axis leaves per-device partial sums
            rules.append(mk(all_gather(src, d), all_reduce(out), True))
        else:
            kept = d - sum(1 for r in dims if r < d)
            rules.append(mk(all_gather(src, d), all_gather(out, kept), True))
    return rules


_OPERATOR_RULES = {
    "Placeholder": lambda n, g: _sources(n),
    "Parameter": lambda n, g: _sources(n),
    "MatMul": _matmul,
    "ElemwiseUnary": _unary,
    "Identity": _unary,
    "ElemwiseBinary": _binary,
    "Reduce": _reduce,
}


def _collectives(ref: str, shape) -> list:
    n = _size(shape)
    rank = len(shape)

    def mk(pre, kind, post, axis=None, axis2=None):
        return _triple((pre,), Instruction(kind, ref, operands=(dist_id(ref, pre),),
                                           output=dist_id(ref, post), axis=axis, axis2=axis2,
                                           elements=n), {post})

    rules = [mk(all_reduce(ref), "all_reduce", identity(ref))]
    rules += [mk(all_reduce(ref), "reduce_scatter", all_gather(ref, d), axis=d) for d in range(rank)]
    rules += [mk(all_gather(ref, d), "all_gather", identity(ref), axis=d) for d in range(rank)]
    # same contract as all_gather; the cost model tells them apart under skew
    rules += [mk(all_gather(ref, d), "grouped_broadcast", identity(ref), axis=d) for d in range(rank)]
    rules += [mk(all_gather(ref, d1), "all_to_all", all_gather(ref, d2), axis=d1, axis2=d2)
              for d1 in range(rank) for d2 in range(rank) if d1 != d2]
    return rules


def derive_theory(g: Graph, m: int) -> Theory:
    """Every sound triple of ``g`` (independent of m; zero-size shards are legal)."""
    if m < 1:
        raise ValueError(f"device count must be >= 1, got {m}")
    triples = []
    for node in g.nodes:
        triples.extend(_OPERATOR_RULES[node.op](node, g))
    for node in g.nodes:
        triples.extend(_collectives(node.id, node.shape))
    for t in triples:
        assert t.post - t.pre, f"vacuous rule derived: {t}"
    sources = frozenset(n.id for n in g.nodes if n.op in ("Placeholder", "Parameter"))
    return Theory(triples=tuple(triples), loss=g.loss, tensor_ids=g.tensor_ids, source_ids=sources,
                  shapes={n.id: n.shape for n in g.nodes})


def fuse_empty_preconditions(t: Theory) -> Theory:
    """Fold each consumed empty-precondition triple T1 into its consumers T2
    (post(T1) ⊆ pre(T2)) as {pre(T2) - post(T1)} [T1;T2] {post(T1) ∪ post(T2)},
    one triple at a time in list order, until none has a consumer."""
    rules = list(t.triples)
    known = {(r.instrs, r.pre, r.post) for r in rules}
    progress = True
    while progress:
        progress = False
        for r in rules:
            if r.pre:
                continue
            users = [c for c in rules if c is not r and r.post <= c.pre]
            if not users:
                continue
            rules.remove(r)
            for c in users:
                fused = HoareTriple(c.pre - r.post, r.instrs + c.instrs, r.post | c.post)
                key = (fused.instrs, fused.pre, fused.post)
                if key not in known:
                    known.add(key)
                    rules.append(fused)
            progress = True
            break
    return replace(t, triples=tuple(rules))


def add_communication_guards(t: Theory) -> Theory:
    """At most one collective per tensor, none on sources: collective triples
    on e need NotComm(e) and grant Comm(e); every state starts NotComm(*)."""
    if not any(i.is_comm for r in t.triples for i in r.instrs):
        return t
    rules = []
    for r in t.triples:
        refs = [i.ref for i in r.instrs if i.is_comm]
        if any(ref in t.source_ids for ref in refs):
            continue
        if refs:
            rules.append(replace(r, pre=r.pre | {not_communicated(x) for x in refs},
                                 post=r.post | {communicated(x) for x in refs}))
        else:
            rules.append(r)
    start = frozenset(not_communicated(ref) for ref in t.tensor_ids)
    return replace(t, triples=tuple(rules), initial_props=start)


def build_theory(g: Graph, m: int, *, guards: bool = True, fuse: bool = True) -> Theory:
    t = derive_theory(g, m)
    if guards:
        t = add_communication_guards(t)
    if fuse:
        t = fuse_empty_preconditions(t)
    return t


def theory_to_json(t: Theory) -> list:
    return [{"pre": sorted(str(p) for p in r.pre), "instrs": [i.to_json() for i in r.instrs],
             "post": sorted(str(p) for p in r.post)} for r in t.triples]
