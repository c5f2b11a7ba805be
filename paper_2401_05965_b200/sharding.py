"""Integer shard extents from ratio rows (reference load_balancer.py:314 and
interpreter.py:205).

Device j owns the contiguous slice [sum(sizes[:j]), sum(sizes[:j+1])) of a
sharded axis; zero-size shards are legal.  The executor derives every buffer
shape and every collective's per-rank element count from these sizes, so
they must match the reference exactly.
"""
from __future__ import annotations

import math


def round_shards(extent: int, ratios) -> list[int]:
    """Nearest-integer shard sizes repaired to sum to ``extent`` one unit at a
    time where the move costs least L1 accuracy (ties to the higher device
    index); never negative."""
    if extent < 0:
        raise ValueError("extent must be nonnegative")
    targets = [extent * r for r in ratios]
    sizes = [math.floor(t + 0.5) for t in targets]
    gap = extent - sum(sizes)
    while gap:
        step = 1 if gap > 0 else -1
        pick, pick_cost = -1, math.inf
        for j, (s, t) in enumerate(zip(sizes, targets)):
            if step < 0 and s == 0:
                continue
            cost = abs(s + step - t) - abs(s - t)
            if cost < pick_cost - 1e-12 or (cost <= pick_cost + 1e-12 and j > pick):
                pick_cost = min(pick_cost, cost)
                pick = j
        sizes[pick] += step
        gap -= step
    return sizes


def build_shard_table(g, B, assignment) -> dict[tuple[str, int], list[int]]:
    """Sizes for every (tensor, axis) from the tensor's segment row."""
    table = {}
    for t in g.tensors.values():
        row = B.row(assignment.row_index(t.id))
        for axis, extent in enumerate(t.shape):
            table[(t.id, axis)] = round_shards(extent, row)
    return table


def table_from_plan(doc: dict) -> dict[tuple[str, int], list[int]]:
    """Shard table of a plan document ({"ref:axis": sizes})."""
    out = {}
    for key, sizes in doc["shard_table"].items():
        ref, _, axis = key.rpartition(":")
        out[(ref, int(axis))] = [int(s) for s in sizes]
    return out


def offsets(sizes) -> list[int]:
    out = [0]
    for s in sizes:
        out.append(out[-1] + s)
    return out
