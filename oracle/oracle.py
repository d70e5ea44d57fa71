"""ctypes front-end of the C oracle (oracle/leo_oracle.c).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg; never by the product package.

`run(ks, prof, cfg)` returns an `OracleResult` of numpy arrays holding the
reference's outputs for one kernel: base edges (build_graph depgraph.py:507),
pruned edges + valid paths (run_pruning analysis.py:302), blame entries
(attribute_blame analysis.py:431), diagnostics, slice levels and line totals.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

from paper_2604_20032_b200 import abi  # noqa: E402

LIB_PATH = HERE / "liboracle.so"


class OracleOut(C.Structure):
    P = C.c_void_p
    _fields_ = [
        ("n_edges", C.c_int32), ("n_regular", C.c_int32),
        ("prod", P), ("cons", P), ("meta", P),
        ("np_edges", C.c_int32),
        ("p_prod", P), ("p_cons", P), ("p_src", P), ("p_meta", P),
        ("p_npaths", P), ("p_first", P), ("p_dist", P),
        ("n_paths", C.c_int32), ("path_len", P), ("path_acc", P),
        ("n_diags", C.c_int32), ("diags", P),
        ("n_entries", C.c_int32),
        ("e_stalled", P), ("e_edge", P), ("e_sub", P), ("e_blame", P), ("e_factors", P),
        ("level", P), ("slice_size", C.c_int32),
        ("line_blame", P), ("line_stall", P),
        ("t", C.c_double * 10),
    ]


_lib = None


def build(force: bool = False) -> Path:
    if force or not LIB_PATH.exists() or \
            LIB_PATH.stat().st_mtime < (HERE / "leo_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = C.CDLL(str(LIB_PATH))
        _lib.oracle_run.restype = C.c_int
        _lib.oracle_run.argtypes = [C.POINTER(abi.LeoKernel), C.POINTER(abi.LeoProfile),
                                    C.POINTER(abi.LeoConfig), C.c_int, C.c_void_p, C.c_int32,
                                    C.POINTER(OracleOut)]
        _lib.oracle_free.argtypes = [C.POINTER(OracleOut)]
        _lib.oracle_bin_samples.restype = C.c_int
        _lib.oracle_bin_samples.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_int32, C.c_void_p, C.c_void_p]
        assert _lib.oracle_sizeof_out() == C.sizeof(OracleOut), "OracleOut layout mismatch"
    return _lib


@dataclass
class OracleResult:
    prod: np.ndarray
    cons: np.ndarray
    meta: np.ndarray
    n_regular: int
    p_prod: np.ndarray = None
    p_cons: np.ndarray = None
    p_meta: np.ndarray = None
    p_src: np.ndarray = None
    p_npaths: np.ndarray = None
    p_first: np.ndarray = None
    p_dist: np.ndarray = None
    path_len: np.ndarray = None
    path_acc: np.ndarray = None
    diags: np.ndarray = None          # [n, 6] code, instr, a0, a1, a2, seq
    e_stalled: np.ndarray = None
    e_edge: np.ndarray = None
    e_sub: np.ndarray = None
    e_blame: np.ndarray = None
    e_factors: np.ndarray = None
    level: np.ndarray = None
    line_blame: np.ndarray = None
    line_stall: np.ndarray = None
    times: tuple = ()


def _arr(ptr, n, dtype, shape=None):
    n = int(n)
    if shape is not None:
        n = int(np.prod(shape))
    if n == 0 or not ptr:
        return np.zeros((0,) if shape is None else (0,) + shape[1:], dtype=dtype)
    buf = (C.c_char * (n * np.dtype(dtype).itemsize)).from_address(ptr)
    a = np.frombuffer(buf, dtype=dtype).copy()
    return a.reshape(shape) if shape is not None else a


def _ptrs(obj):
    keep = {}

    def ptr(name):
        a = np.ascontiguousarray(getattr(obj, name))
        keep[name] = a
        return a.ctypes.data
    return ptr, keep


def run(ks, prof, cfg=None, stages: str = "all") -> OracleResult:
    """Run the oracle on one kernel.  stages: "graph", "prune" or "all"."""
    L = lib()
    kptr, kkeep = _ptrs(ks)
    k = abi.kernel_struct(ks, kptr)
    pptr, pkeep = _ptrs(prof)
    p = abi.profile_struct(prof, pptr)
    if cfg is None:
        cfg = abi.make_config(dialect=ks.dialect)
    flags = {"graph": 1, "prune": 3, "all": 31}[stages]
    line_id = np.ascontiguousarray(ks.line_id, dtype=np.int32)
    n_lines = max(len(ks.lines), int(line_id.max()) + 1 if line_id.size else 1)
    out = OracleOut()
    rc = L.oracle_run(C.byref(k), C.byref(p), C.byref(cfg), flags, line_id.ctypes.data,
                      n_lines, C.byref(out))
    if rc != 0:
        raise RuntimeError(f"oracle_run failed: {rc}")
    try:
        r = OracleResult(prod=_arr(out.prod, out.n_edges, np.int32),
                         cons=_arr(out.cons, out.n_edges, np.int32),
                         meta=_arr(out.meta, out.n_edges, np.uint32), n_regular=out.n_regular,
                         diags=_arr(out.diags, out.n_diags, np.int32, (out.n_diags, 6)),
                         times=tuple(out.t))
        if flags & 2:
            n = out.np_edges
            r.p_prod = _arr(out.p_prod, n, np.int32)
            r.p_cons = _arr(out.p_cons, n, np.int32)
            r.p_meta = _arr(out.p_meta, n, np.uint32)
            r.p_src = _arr(out.p_src, n, np.int32)
            r.p_npaths = _arr(out.p_npaths, n, np.int32)
            r.p_first = _arr(out.p_first, n, np.int32)
            r.p_dist = _arr(out.p_dist, n, np.float64)
            r.path_len = _arr(out.path_len, out.n_paths, np.int32)
            r.path_acc = _arr(out.path_acc, out.n_paths, np.float64)
        if flags & 4:
            m = out.n_entries
            r.e_stalled = _arr(out.e_stalled, m, np.int32)
            r.e_edge = _arr(out.e_edge, m, np.int32)
            r.e_sub = _arr(out.e_sub, m, np.uint8)
            r.e_blame = _arr(out.e_blame, m, np.float64)
            r.e_factors = _arr(out.e_factors, m * 4, np.float64, (m, 4))
            r.level = _arr(out.level, ks.n_instr, np.int32)
            r.line_blame = _arr(out.line_blame, n_lines, np.float64)
            r.line_stall = _arr(out.line_stall, n_lines, np.float64)
    finally:
        L.oracle_free(C.byref(out))
    return r


def bin_samples(pc: np.ndarray, cat: np.ndarray, lut: np.ndarray, n_instr: int):
    """Stage-0 restatement: raw (pc, category) stream -> lat[N], cls_cnt[N, 8]."""
    L = lib()
    pc = np.ascontiguousarray(pc, dtype=np.int32)
    cat = np.ascontiguousarray(cat, dtype=np.uint8)
    lut = np.ascontiguousarray(lut, dtype=np.uint8)
    lat = np.zeros(n_instr, dtype=np.int32)
    cls = np.zeros((n_instr, 8), dtype=np.int32)
    rc = L.oracle_bin_samples(pc.shape[0], pc.ctypes.data, cat.ctypes.data, lut.ctypes.data,
                              n_instr, lat.ctypes.data, cls.ctypes.data)
    if rc != 0:
        raise ValueError("sample pc out of range")
    return lat, cls
