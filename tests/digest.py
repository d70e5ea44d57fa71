"""Size-independent golden form of one analysis: per-field SHA-256 digests.

Full-size configs (C2 10k, C3 50k, C5 1M instructions, C4 kernels) are too
large to commit as arrays, so `tests/golden/make_full.py` runs the REFERENCE
on them here and stores, per field, the digest of a canonical byte form plus
its length.  The GPU parity tests (and the oracle tests) compute the same
digests from their own outputs: a match is bit-exact equality of

  base edges (bprod / bcons / bmeta), pruned edges (pprod / pcons / pmeta),
  valid paths (npaths + the records flattened in edge order), diagnostics,
  blame entries (stalled, cause, kind, sub, register, blame cycles, factors),
  slice levels,

while the per-line vectors (device FP64 atomics: summation order differs)
are compared through their sums, non-zero supports and two weighted
checksums within a relative tolerance.
"""

from __future__ import annotations

import hashlib

import numpy as np

EXACT = ("bprod", "bcons", "bmeta", "pprod", "pcons", "pmeta", "npaths", "plen_flat",
         "pacc_flat", "diags", "bl_stalled", "bl_cause", "bl_kind", "bl_sub", "bl_reg",
         "bl_blame", "bl_factors", "level")
LINE_REL = 1e-9


def _flat_paths(x: dict):
    n = np.asarray(x["npaths"], dtype=np.int64)
    first = np.asarray(x["first"], dtype=np.int64)
    plen, pacc = np.asarray(x["plen"]), np.asarray(x["pacc"])
    if n.sum() == 0:
        return np.zeros(0, np.int32), np.zeros(0, np.float64)
    sel = np.flatnonzero(n > 0)
    starts = np.concatenate([[0], np.cumsum(n[sel])[:-1]])     # position of each run in the flat list
    idx = np.repeat(first[sel] - starts, n[sel]) + np.arange(int(n[sel].sum()))
    return plen[idx].astype(np.int32), pacc[idx].astype(np.float64)


def _bytes(name: str, v) -> bytes:
    if name in ("diags", "bl_reg"):
        return "\n".join(str(s) for s in v).encode()
    a = np.asarray(v)
    dt = {"bmeta": np.uint32, "pmeta": np.uint32, "bl_kind": np.uint8, "bl_sub": np.uint8,
          "bl_blame": np.float64, "bl_factors": np.float64, "pacc_flat": np.float64}.get(name, np.int32)
    a = np.ascontiguousarray(a.astype(dt, copy=False))
    if name == "bl_factors":
        a = np.where(np.isnan(a), 0.0, a)              # self entries: no factors
    return a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes()


def _line_checks(v) -> dict:
    v = np.asarray(v, dtype=np.float64)
    rng = np.random.Generator(np.random.PCG64(20260417))
    w = rng.random(v.shape[0])
    idx = np.arange(v.shape[0], dtype=np.float64)
    return {"n": int(v.shape[0]), "nnz": int(np.count_nonzero(v)), "sum": float(v.sum()),
            "wsum": float(np.dot(v, w)), "isum": float(np.dot(v, idx)),
            "support": hashlib.sha256(np.flatnonzero(v).astype(np.int64).tobytes()).hexdigest()}


def digests(x: dict) -> dict:
    """Golden-field arrays (tests/golden_io.py names) -> digest record."""
    y = dict(x)
    y["plen_flat"], y["pacc_flat"] = _flat_paths(x)
    out = {}
    for name in EXACT:
        v = y[name]
        out[name] = {"len": int(len(v)), "sha256": hashlib.sha256(_bytes(name, v)).hexdigest()}
    for name in ("line_blame", "line_stall"):
        out[name] = _line_checks(y[name])
    return out


def compare(exp: dict, got: dict, line_rel: float = LINE_REL) -> list[str]:
    errs = []
    for name in EXACT:
        if exp[name] != got[name]:
            errs.append(f"{name}: {got[name]} != reference {exp[name]}")
    for name in ("line_blame", "line_stall"):
        a, b = exp[name], got[name]
        if (a["n"], a["nnz"], a["support"]) != (b["n"], b["nnz"], b["support"]):
            errs.append(f"{name}: support differs ({b['nnz']} vs {a['nnz']} non-zero lines)")
        for k in ("sum", "wsum", "isum"):
            if abs(a[k] - b[k]) > line_rel * max(abs(a[k]), 1.0):
                errs.append(f"{name}.{k}: {b[k]!r} != reference {a[k]!r}")
    return errs
