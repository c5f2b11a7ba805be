"""Distributed-program vocabulary shared by the planner and the B200 executor.

Mirrors the reference's instruction set and naming so that plan documents
written by either side load on the other (reference: theory.py:27-155,
synthesizer.py:53-70):

* a *property* ``e|F`` says the per-device instances of a distributed tensor
  reconstruct the reference tensor ``e`` under form ``F`` — ``Id`` (every
  device holds ``e``), ``AG(d)`` (concatenate along axis ``d``) or ``AR``
  (elementwise sum over devices);
* a distributed tensor is named ``e@full``, ``e@shard<d>`` or ``e@partial``;
* an instruction runs on every device in lock step.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

IDENTITY = "Id"
ALL_GATHER = "AG"
ALL_REDUCE = "AR"
COMMUNICATED = "Comm"
NOT_COMMUNICATED = "NotComm"
GUARD_KINDS = (COMMUNICATED, NOT_COMMUNICATED)

COMM_KINDS = ("all_reduce", "all_gather", "reduce_scatter", "all_to_all", "grouped_broadcast")
SOURCE_KINDS = ("placeholder", "placeholder_shard", "parameter", "parameter_shard")
COMPUTE_KINDS = ("matmul", "elemwise_unary", "elemwise_binary", "reduce", "identity")


@dataclass(frozen=True)
class Property:
    ref: str
    kind: str
    axis: int | None = None

    @property
    def is_guard(self) -> bool:
        return self.kind in GUARD_KINDS

    def __str__(self) -> str:
        return f"{self.ref}|AG({self.axis})" if self.kind == ALL_GATHER else f"{self.ref}|{self.kind}"


def identity(ref: str) -> Property:
    return Property(ref, IDENTITY)


def all_gather(ref: str, d: int) -> Property:
    return Property(ref, ALL_GATHER, d)


def all_reduce(ref: str) -> Property:
    return Property(ref, ALL_REDUCE)


def communicated(ref: str) -> Property:
    return Property(ref, COMMUNICATED)


def not_communicated(ref: str) -> Property:
    return Property(ref, NOT_COMMUNICATED)


_SUFFIX = {IDENTITY: "full", ALL_REDUCE: "partial"}


def dist_id(ref: str, prop: Property) -> str:
    """Name of the distributed tensor realising ``prop`` (theory.py:77)."""
    if prop.kind == ALL_GATHER:
        return f"{ref}@shard{prop.axis}"
    if prop.kind in _SUFFIX:
        return f"{ref}@{_SUFFIX[prop.kind]}"
    raise ValueError(f"guard property {prop} has no distributed tensor")


def form_of_dist_id(did: str) -> Property:
    """Inverse of :func:`dist_id` (theory.py:88)."""
    ref, _, suffix = did.rpartition("@")
    if suffix == "full":
        return identity(ref)
    if suffix == "partial":
        return all_reduce(ref)
    if suffix.startswith("shard"):
        return all_gather(ref, int(suffix[5:]))
    raise ValueError(f"malformed distributed tensor id {did!r}")


@dataclass(frozen=True)
class Instruction:
    """One SPMD instruction (theory.py:99).  ``sharded`` says whether the
    per-device work scales with the device's ratio; ``elements`` is the
    reference-tensor size a collective moves (0 for compute)."""
    kind: str
    ref: str
    operands: tuple[str, ...] = ()
    output: str = ""
    axis: int | None = None
    axis2: int | None = None
    dims: tuple[int, ...] | None = None
    tag: str | None = None
    sharded: bool = False
    flops: int = 0
    elements: int = 0

    @property
    def is_comm(self) -> bool:
        return self.kind in COMM_KINDS

    def canonical(self) -> str:
        parts = [self.kind, self.ref]
        if self.axis is not None:
            parts.append(f"d={self.axis}")
        if self.axis2 is not None:
            parts.append(f"d2={self.axis2}")
        return f"{self.output}<-{'/'.join(parts)}({','.join(self.operands)})"

    def to_json(self) -> dict:
        doc: dict = {"kind": self.kind, "ref": self.ref, "operands": list(self.operands),
                     "output": self.output}
        for key in ("axis", "axis2"):
            if getattr(self, key) is not None:
                doc[key] = getattr(self, key)
        if self.dims is not None:
            doc["dims"] = list(self.dims)
        if self.tag is not None:
            doc["tag"] = self.tag
        doc.update(sharded=self.sharded, flops=self.flops, elements=self.elements)
        return doc

    @classmethod
    def from_json(cls, doc: dict) -> "Instruction":
        dims = doc.get("dims")
        return cls(kind=doc["kind"], ref=doc["ref"], operands=tuple(doc.get("operands", ())),
                   output=doc["output"], axis=doc.get("axis"), axis2=doc.get("axis2"),
                   dims=None if dims is None else tuple(dims), tag=doc.get("tag"),
                   sharded=doc["sharded"], flops=doc["flops"], elements=doc["elements"])


@dataclass(frozen=True)
class DistributedProgram:
    """A complete program plus the loss it realises (synthesizer.py:53)."""
    instrs: tuple[Instruction, ...]
    loss: str

    def canonical(self) -> str:
        return ";".join(i.canonical() for i in self.instrs)

    def fingerprint(self) -> str:
        return hashlib.sha256(self.canonical().encode()).hexdigest()

    def to_json(self) -> dict:
        return {"loss": self.loss, "instrs": [i.to_json() for i in self.instrs]}

    @classmethod
    def from_json(cls, doc: dict) -> "DistributedProgram":
        return cls(instrs=tuple(Instruction.from_json(d) for d in doc["instrs"]), loss=doc["loss"])
