"""Output types of the drop-in API.

When the caller passes `stalltrace` objects, results are built from the
reference's own classes (so equality with the reference holds).  Otherwise
these mirrors are used: same class names, field names and enum values as
depgraph.py:46-122 and analysis.py:320-368, so code written against the
reference reads them unchanged.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

from . import enums as E


class RegClass(enum.Enum):
    VECTOR_GPR = "vector_gpr"
    SCALAR_GPR = "scalar_gpr"
    PREDICATE = "predicate"
    BARRIER = "barrier"
    UNIFORM = "uniform"
    SBID_TOKEN = "sbid_token"
    SPECIAL = "special"


class EdgeKind(enum.Enum):
    RAW = "raw"
    GUARD = "guard"
    MEM_WAITCNT = "mem_waitcnt"
    MEM_BARRIER = "mem_barrier"
    MEM_SWSB = "mem_swsb"


class DepClass(enum.Enum):
    MEMORY = "memory"
    EXECUTION = "execution"
    SYNCHRONIZATION = "synchronization"


class SelfBlame(enum.Enum):
    MEMORY_LATENCY = "memory_latency"
    COMPUTE_SATURATION = "compute_saturation"
    SYNCHRONIZATION_OVERHEAD = "synchronization_overhead"
    PIPELINE_CONTENTION = "pipeline_contention"
    INSTRUCTION_FETCH = "instruction_fetch"
    INDIRECT_ADDRESSING = "indirect_addressing"


assert tuple(c.value for c in RegClass) == E.REG_CLASSES
assert tuple(c.value for c in EdgeKind) == E.EDGE_KINDS
assert tuple(c.value for c in DepClass) == E.DEP_CLASSES
assert tuple(c.value for c in SelfBlame) == E.SELF_BLAMES


@dataclass(frozen=True)
class RegisterRef:
    reg_class: RegClass
    index: int
    span: int = 1


@dataclass(frozen=True)
class PathRecord:
    length_instructions: int
    accumulated_issue_cycles: float


@dataclass(frozen=True)
class DepEdge:
    producer: int
    consumer: int
    kind: EdgeKind
    register: RegisterRef | None
    dep_class: DepClass
    valid_paths: tuple = ()


class DependencyGraph:
    """Edge list plus per-node adjacency in edge-list order (depgraph.py:94-122)."""

    def __init__(self, attached, edges, diagnostics=()):
        self.attached = attached
        self.edges = tuple(edges)
        self.diagnostics = tuple(diagnostics)
        inc: dict[int, list[int]] = {}
        out: dict[int, list[int]] = {}
        for i, e in enumerate(self.edges):
            inc.setdefault(e.consumer, []).append(i)
            out.setdefault(e.producer, []).append(i)
        self.incoming = {k: tuple(v) for k, v in inc.items()}
        self.outgoing = {k: tuple(v) for k, v in out.items()}

    @property
    def cfg(self):
        return self.attached.cfg

    def incoming_edges(self, node):
        return [self.edges[i] for i in self.incoming.get(node, ())]

    def outgoing_edges(self, node):
        return [self.edges[i] for i in self.outgoing.get(node, ())]

    def with_edges(self, edges, extra_diagnostics=()):
        return DependencyGraph(self.attached, edges, self.diagnostics + tuple(extra_diagnostics))


@dataclass(frozen=True)
class Factors:
    dist: float
    eff: float
    isu: float
    match: float

    @property
    def product(self) -> float:
        return self.dist * self.eff * self.isu * self.match


@dataclass(frozen=True)
class BlameEntry:
    stalled: int
    cause: int | None
    kind: EdgeKind | None
    subcategory: SelfBlame | None
    blame_cycles: float
    factors: Factors | None
    register: str | None = None


@dataclass(frozen=True)
class UseLink:
    producer: int
    consumer: int
    register: RegisterRef
    kind: EdgeKind


@dataclass(frozen=True)
class ChainHop:
    index: int
    kind: EdgeKind | None
    blame_cycles: float | None
    share: float | None
    self_blame: SelfBlame | None


@dataclass(frozen=True)
class Coverage:
    value: float
    vacuous: bool


class Namespace:
    """The set of output classes to construct (reference's or mirrors)."""

    def __init__(self, **kw):
        self.__dict__.update(kw)

    @classmethod
    def mirror(cls):
        return cls(RegClass=RegClass, EdgeKind=EdgeKind, DepClass=DepClass, SelfBlame=SelfBlame,
                   RegisterRef=RegisterRef, PathRecord=PathRecord, DepEdge=DepEdge,
                   DependencyGraph=DependencyGraph, Factors=Factors, BlameEntry=BlameEntry,
                   UseLink=UseLink, ChainHop=ChainHop, Coverage=Coverage)

    @classmethod
    def from_modules(cls, depgraph, analysis, isa):
        return cls(RegClass=isa.RegClass, EdgeKind=depgraph.EdgeKind, DepClass=depgraph.DepClass,
                   SelfBlame=analysis.SelfBlame, RegisterRef=isa.RegisterRef,
                   PathRecord=depgraph.PathRecord, DepEdge=depgraph.DepEdge,
                   DependencyGraph=depgraph.DependencyGraph, Factors=analysis.Factors,
                   BlameEntry=analysis.BlameEntry, UseLink=depgraph.UseLink,
                   ChainHop=analysis.ChainHop, Coverage=analysis.Coverage)
