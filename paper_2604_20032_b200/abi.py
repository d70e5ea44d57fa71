"""ctypes mirror of include/leo_b200.h (structs only; no library loading).

Shared by the device wrapper (`_lib.py`, device pointers) and the oracle
wrapper in oracle/ (host pointers)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import enums as E

P = C.c_void_p


class LeoKernel(C.Structure):
    _fields_ = [
        ("n_instr", C.c_int32), ("n_blocks", C.c_int32), ("n_units", C.c_int32),
        ("dialect", C.c_int32), ("n_opnd", C.c_int32), ("n_use_units", C.c_int32),
        ("n_def_units", C.c_int32), ("unit_base", C.c_int32 * 8),
        ("opclass", P), ("block_of", P), ("opnd_ptr", P), ("opnd", P),
        ("sync_kind", P), ("sync_a", P), ("sync_b", P),
        ("blk_first", P), ("blk_last", P), ("succ_ptr", P), ("succ", P),
        ("pred_ptr", P), ("pred", P),
        ("n_segments", C.c_int32), ("max_seg_blocks", C.c_int32), ("seg_block", P),
    ]


class LeoProfile(C.Structure):
    _fields_ = [
        ("period", C.c_int64), ("lat", P), ("cls_cnt", P), ("exec_cnt", P),
        ("total", P), ("eff", P), ("sampled", P),
    ]


class LeoSamples(C.Structure):
    _fields_ = [("n_samples", C.c_int64), ("pc", P), ("cat", P), ("cat_to_cs", P),
                ("pc_host", P), ("cat_host", P), ("packed", P), ("packed_host", P),
                ("packed_bytes", C.c_int32), ("packed_cat_bits", C.c_int32)]


class LeoConfig(C.Structure):
    _fields_ = [
        ("stage_mask", C.c_uint32), ("prune_exec", C.c_int32), ("max_paths", C.c_int32),
        ("max_depth", C.c_int32), ("threshold", C.c_double * 16),
        ("consumer_lo", C.c_int32), ("consumer_hi", C.c_int32),
    ]


class LeoTrace(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("count", C.c_int32), ("only_kernel", C.c_int32),
                ("mode", C.c_int32), ("ev_begin", P), ("ev_end", P), ("kernel_id", P)]


class LeoCaps(C.Structure):
    _fields_ = [("query_results", C.c_int64), ("candidates", C.c_int64),
                ("sync_keys", C.c_int64), ("slow_items", C.c_int64),
                ("trace", C.POINTER(LeoTrace)), ("debug_flags", C.c_int32), ("options", C.c_int32),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_int64),
                ("workspace_needed", C.POINTER(C.c_int64))]


DBG_REACH_T2, DBG_REACH_T3, DBG_SYNC_SLOW, DBG_PRUNE_SLOW, DBG_SELF_SLOW, DBG_NO_SMEM = 1, 2, 4, 8, 16, 32
DBG_PHASES = 64
OPT_ACCUMULATE_LINES = 1


class LeoEdges(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("prod", P), ("cons", P), ("meta", P),
                ("count", P), ("n_regular", P)]


class LeoPaths(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("first", P), ("npaths", P), ("dist", P),
                ("len", P), ("accum", P), ("count", P)]


class LeoDiag(C.Structure):
    _fields_ = [("code", C.c_int32), ("instr", C.c_int32), ("a0", C.c_int32),
                ("a1", C.c_int32), ("a2", C.c_int32), ("seq", C.c_int32)]


class LeoDiags(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("rec", P), ("count", P)]


class LeoBlame(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("stalled", P), ("edge", P), ("sub", P),
                ("blame", P), ("factors", P), ("count", P), ("cause", P), ("meta", P)]


class LeoReport(C.Structure):
    _fields_ = [("top_n", C.c_int32), ("include_unsampled", C.c_int32), ("chain_depth", C.c_int32),
                ("max_causes", C.c_int32), ("coverage", P), ("n_hot", P), ("hot", P),
                ("n_causes", P), ("causes", P), ("chain_len", P), ("chain_node", P),
                ("chain_entry", P), ("chain_self", P)]


class LeoReachIn(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("set_off", P), ("defs", P), ("count", P)]


DIAG_UNRESOLVED, DIAG_WAITCNT, DIAG_NO_SETTER, DIAG_PATH_CAPPED = 1, 2, 3, 4
ST_EDGE_OVERFLOW, ST_PATH_OVERFLOW, ST_DIAG_OVERFLOW = 1, 2, 4
ST_BLAME_OVERFLOW, ST_SCRATCH_OVERFLOW, ST_BAD_INPUT = 8, 16, 32


def make_config(stage_mask=(1, 2, 3, 4), prune_exec=False, max_paths=64, max_depth=512,
                thresholds=None, dialect="nvidia", consumer_range=None) -> LeoConfig:
    cfg = LeoConfig()
    if consumer_range is not None:
        cfg.consumer_lo, cfg.consumer_hi = int(consumer_range[0]), int(consumer_range[1])
    m = 0
    for s in stage_mask:
        if 1 <= int(s) <= 4:
            m |= 1 << (int(s) - 1)
    cfg.stage_mask = m
    cfg.prune_exec = 1 if prune_exec else 0
    cfg.max_paths = int(max_paths)
    cfg.max_depth = int(max_depth)
    th = thresholds if thresholds is not None else E.default_thresholds(dialect)
    for i, v in enumerate(th):
        cfg.threshold[i] = float(v)
    return cfg


def config_from_reference(config, dialect: str) -> LeoConfig:
    """Translate a reference `AnalysisConfig` (analysis.py:115-124), duck-typed."""
    table = config.latency
    if table is None:
        th = E.default_thresholds(dialect)
    else:
        th = E.dense_thresholds((c.value, v) for c, v in table.thresholds)
    return make_config(config.stage_mask, config.prune_exec, config.max_paths,
                       config.max_depth, th, dialect)


def kernel_struct(ks, ptr) -> LeoKernel:
    """Fill a LeoKernel whose array fields come from `ptr(name) -> address`."""
    k = LeoKernel()
    k.n_instr = ks.n_instr
    k.n_blocks = ks.n_blocks
    k.n_units = ks.n_units
    k.dialect = ks.dialect_idx
    k.n_opnd = int(ks.opnd.shape[0])
    use_units, def_units = unit_counts(ks)
    k.n_use_units = use_units
    k.n_def_units = def_units
    for c in range(8):
        k.unit_base[c] = int(ks.unit_base[c])
    for name in ("opclass", "block_of", "opnd_ptr", "opnd", "sync_kind", "sync_a", "sync_b",
                 "blk_first", "blk_last", "succ_ptr", "succ", "pred_ptr", "pred"):
        setattr(k, name, ptr(name))
    sb = getattr(ks, "seg_block", None)
    if sb is not None and len(sb) > 2:
        k.n_segments = len(sb) - 1
        k.max_seg_blocks = int(np.diff(np.asarray(sb)).max())
        k.seg_block = ptr("seg_block")
    return k


def unit_counts(ks) -> tuple[int, int]:
    """(sum of spans over src+guard operands, over dest operands)."""
    import numpy as np
    op = np.asarray(ks.opnd, dtype=np.uint32)
    span = ((op >> 16) & 0xFF).astype(np.int64)
    dst = ((op >> 27) & 3) == E.ROLE_DST
    return int(span[~dst].sum()), int(span[dst].sum())


def profile_struct(prof, ptr) -> LeoProfile:
    p = LeoProfile()
    p.period = int(prof.period)
    for name in ("lat", "cls_cnt", "exec_cnt", "total", "eff", "sampled"):
        setattr(p, name, ptr(name))
    return p
