"""Loaders for the committed golden fixtures (tests/golden/, made by make_golden.py
from the reference package)."""
from __future__ import annotations

import glob
import hashlib
import json
import os

import numpy as np

from paper_2401_05965_b200 import graph_ir, workloads

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_json(*parts):
    with open(os.path.join(GOLDEN, *parts), encoding="utf-8") as fh:
        return json.load(fh)


def graph_doc(name: str) -> dict:
    if name.startswith("bert12_b"):
        return workloads.bert_doc(layers=12, batch=int(name[len("bert12_b"):]), seq=128)
    if name.startswith("moe12_b"):
        return workloads.moe_stack_doc(layers=12, batch=int(name[len("moe12_b"):]), seq=128)
    return load_json("graphs", f"{name}.json")


def graph(name: str):
    return graph_ir.graph_from_dict(graph_doc(name))


def plan(gname: str, cname: str) -> dict:
    return load_json("plans", f"{gname}.{cname}.json")


def value_cases() -> list[tuple[str, str]]:
    out = []
    for path in sorted(glob.glob(os.path.join(GOLDEN, "values", "*.npz"))):
        stem = os.path.basename(path)[:-4]
        gname, cname = stem.rsplit(".", 1)
        out.append((gname, cname))
    return out


def values(gname: str, cname: str):
    return np.load(os.path.join(GOLDEN, "values", f"{gname}.{cname}.npz"))


def seeds(vals) -> list[int]:
    return sorted({int(k.split(":")[0][4:]) for k in vals.files if k.startswith("seed")})


def _sha(value) -> str:
    return hashlib.sha256(np.ascontiguousarray(value, dtype=np.float64).tobytes()).hexdigest()


def inputs(g, vals, seed: int) -> dict:
    """The exact float64 inputs the reference was run on (regenerated from the
    seed when not stored verbatim; the stored SHA-256 guards against drift)."""
    stored = {k.split(":", 2)[2]: vals[k] for k in vals.files if k.startswith(f"seed{seed}:input:")}
    if stored:
        return stored
    out = workloads.synthetic_inputs(g, seed, scaled=bool(vals["scaled"]))
    for name, value in out.items():
        want = str(vals[f"seed{seed}:sha:{name}"])
        if _sha(value) != want:
            raise AssertionError(f"regenerated input {name!r} differs from the golden run")
    return out


def env(vals) -> dict:
    """Reference interpreter env (seed 0): {did: [per-device arrays]}."""
    out: dict = {}
    for key in vals.files:
        if key.startswith("env:"):
            _, did, dev = key.split(":")
            out.setdefault(did, {})[int(dev)] = vals[key]
    return {did: [d[j] for j in sorted(d)] for did, d in out.items()}


def program_cases() -> list[str]:
    """Enumerated programs WITH collectives (tests/golden/programs/)."""
    return sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(GOLDEN, "programs", "*.json")))


def program_case(stem: str):
    doc = load_json("programs", f"{stem}.json")
    vals = np.load(os.path.join(GOLDEN, "programs", f"{stem}.npz"))
    return doc, vals, stem.split(".")[0]
