"""Enumeration orders shared by the host mirror, the SoA encoder, the C oracle
and the CUDA kernels.

Every index below follows the definition order of the reference enum it
mirrors (the reference uses enum *string values* for sorting; the tables at the
bottom reproduce those string orders as integer ranks).

Reference enums:
  Dialect       isa.py:19-22        RegClass     isa.py:32-39
  OpcodeClass   isa.py:42-58        CommonStall  profile.py:29-43
  EdgeKind      depgraph.py:46-51   DepClass     depgraph.py:57-60
  SelfBlame     analysis.py:320-326
"""

from __future__ import annotations

DIALECTS = ("nvidia", "amd", "intel")
REG_CLASSES = ("vector_gpr", "scalar_gpr", "predicate", "barrier", "uniform",
               "sbid_token", "special")
OPCODE_CLASSES = ("global_load", "global_store", "local_load", "local_store",
                  "scalar_load", "constant_load", "atomic", "fp_arith", "int_arith",
                  "conversion", "control_flow", "sync_wait", "barrier_all", "send",
                  "nop", "other")
COMMON_STALLS = ("memory_dep", "execution_dep", "synchronization", "instruction_fetch",
                 "pipeline_busy", "not_selected", "idle", "other")
EDGE_KINDS = ("raw", "guard", "mem_waitcnt", "mem_barrier", "mem_swsb")
DEP_CLASSES = ("memory", "execution", "synchronization")
SELF_BLAMES = ("memory_latency", "compute_saturation", "synchronization_overhead",
               "pipeline_contention", "instruction_fetch", "indirect_addressing")
SYNC_NONE, SYNC_WAITCNT, SYNC_BARRIER, SYNC_SWSB = 0, 1, 2, 3

DIALECT_IDX = {v: i for i, v in enumerate(DIALECTS)}
RC_IDX = {v: i for i, v in enumerate(REG_CLASSES)}
OC_IDX = {v: i for i, v in enumerate(OPCODE_CLASSES)}
CS_IDX = {v: i for i, v in enumerate(COMMON_STALLS)}
EK_IDX = {v: i for i, v in enumerate(EDGE_KINDS)}
DC_IDX = {v: i for i, v in enumerate(DEP_CLASSES)}
SB_IDX = {v: i for i, v in enumerate(SELF_BLAMES)}

ROLE_SRC, ROLE_GUARD, ROLE_DST = 0, 1, 2
NONE_U32 = 0xFFFFFFFF

# RegClass rank in `.value` string order, used by the build_graph sort key
# (depgraph.py:514-516): barrier < predicate < scalar_gpr < sbid_token <
# special < uniform < vector_gpr.
RC_SORT_RANK = tuple(sorted(REG_CLASSES).index(c) for c in REG_CLASSES)

# class sets (isa.py:61-85)
LOAD_CLASSES = frozenset(OC_IDX[c] for c in ("global_load", "local_load", "scalar_load",
                                             "constant_load"))
MEMORY_PRODUCER_CLASSES = LOAD_CLASSES | {OC_IDX["atomic"], OC_IDX["send"]}
COMPUTE_CLASSES = frozenset(OC_IDX[c] for c in ("fp_arith", "int_arith", "conversion"))
STORE_CLASSES = frozenset(OC_IDX[c] for c in ("global_store", "local_store"))
MEMORY_CLASSES = MEMORY_PRODUCER_CLASSES | STORE_CLASSES
VMCNT_CLASSES = frozenset(OC_IDX[c] for c in ("global_load", "global_store", "atomic"))
LGKMCNT_CLASSES = frozenset(OC_IDX[c] for c in ("local_load", "local_store", "scalar_load",
                                                "constant_load"))

# Per-dialect vendor stall categories -> CommonStall (profile.py:52-99).  The
# category id used by the raw-sample stream is the position in the sorted
# category list (`vendor_categories`, profile.py:102-103).
_NVIDIA_MAP = {
    "instruction fetch": "instruction_fetch", "execution dependency": "execution_dep",
    "memory dependency": "memory_dep", "texture": "memory_dep",
    "synchronization": "synchronization", "constant memory dependency": "memory_dep",
    "pipe busy": "pipeline_busy", "memory throttle": "memory_dep",
    "not selected": "not_selected", "sleeping": "idle", "other": "other",
}
_AMD_MAP = {
    "no instruction available": "instruction_fetch", "alu dependency": "execution_dep",
    "waiting for memory": "memory_dep", "internal instruction": "other",
    "barrier wait": "synchronization", "not selected": "not_selected",
    "pipeline stall": "pipeline_busy", "sleep": "idle", "other": "other",
}
_INTEL_MAP = {
    "control flow": "other", "control flow stalls": "other", "controlstall": "other",
    "pipeline hazards": "execution_dep", "pipestall": "execution_dep",
    "memory send operations": "memory_dep", "sendstall": "memory_dep",
    "scoreboard id dependencies": "synchronization", "sbidstall": "synchronization",
    "synchronization": "synchronization", "syncstall": "synchronization",
    "instruction fetch": "instruction_fetch", "instrfetchstall": "instruction_fetch",
    "distribution stalls": "pipeline_busy", "diststall": "pipeline_busy",
    "other stalls": "other", "otherstall": "other",
}
STALL_MAPS = {"nvidia": _NVIDIA_MAP, "amd": _AMD_MAP, "intel": _INTEL_MAP}


def vendor_categories(dialect: str) -> tuple[str, ...]:
    """Sorted vendor category names (profile.py:102-103); index = category id."""
    return tuple(sorted(STALL_MAPS[dialect]))


def category_lut(dialect: str):
    """uint8[256] vendor-category-id -> CommonStall index."""
    import numpy as np
    lut = np.full(256, CS_IDX["other"], dtype=np.uint8)
    for i, name in enumerate(vendor_categories(dialect)):
        lut[i] = CS_IDX[STALL_MAPS[dialect][name]]
    return lut


def norm_category(category: str) -> str:
    """profile.py:46-47"""
    return " ".join(category.lower().split())


# Default latency tables (analysis.py:55-82); units cycles (nvidia) or
# instructions (amd/intel).
NVIDIA_LATENCY = {
    "global_load": 200.0, "global_store": 200.0, "atomic": 200.0, "send": 200.0,
    "local_load": 30.0, "local_store": 30.0, "scalar_load": 30.0, "constant_load": 20.0,
    "fp_arith": 6.0, "int_arith": 4.0, "conversion": 6.0, "other": 6.0,
}
COUNT_LATENCY = {
    "global_load": 32.0, "global_store": 32.0, "atomic": 32.0, "send": 32.0,
    "local_load": 8.0, "local_store": 8.0, "scalar_load": 8.0, "constant_load": 8.0,
    "fp_arith": 2.0, "int_arith": 2.0, "conversion": 2.0, "other": 2.0,
}


def dense_thresholds(items) -> list[float]:
    """LatencyTable.get for every OpcodeClass (analysis.py:98-104): listed
    classes take their value, every other class falls back to the max."""
    items = list(items)
    fallback = max(v for _, v in items)
    table = {}
    for c, v in items:
        table.setdefault(c, v)   # `get` returns the first match
    return [float(table.get(c, fallback)) for c in OPCODE_CLASSES]


def default_thresholds(dialect: str) -> list[float]:
    src = NVIDIA_LATENCY if dialect == "nvidia" else COUNT_LATENCY
    return dense_thresholds(src.items())
