"""Parity comparator shared by the oracle tests and the GPU parity tests.

`got` and `exp` are dicts of arrays using the golden field names
(tests/golden_io.py).  Edges, pruned edges, valid paths, diagnostics, slice
levels and blame structure are compared bit-exactly; blame cycles and
factors within `rel` (north star: 1e-6 relative; the oracle and the device
reproduce CPython's float arithmetic, so tests pass rel=0 where stated);
line totals within `line_rel` (their summation order differs on the device).
"""

from __future__ import annotations

import numpy as np


def _paths(d, x):
    n = int(d["npaths"][x])
    if n == 0:
        return ()
    f = int(d["first"][x])
    return tuple(zip(d["plen"][f:f + n].tolist(), d["pacc"][f:f + n].tolist()))


def compare(exp: dict, got: dict, rel: float = 0.0, line_rel: float = 1e-9,
            parts=("base", "pruned", "diags", "blame", "slice", "lines")) -> list[str]:
    errs = []

    def eq(name):
        a, b = np.asarray(exp[name]), np.asarray(got[name])
        if a.shape != b.shape or not np.array_equal(a, b):
            bad = "shape" if a.shape != b.shape else int(np.flatnonzero(a.ravel() != b.ravel())[0])
            errs.append(f"{name}: mismatch ({a.shape} vs {b.shape}; first bad {bad})")
            return False
        return True

    if "base" in parts:
        for f in ("bprod", "bcons", "bmeta"):
            eq(f)
    if "pruned" in parts:
        ok = all([eq("pprod"), eq("pcons"), eq("pmeta"), eq("npaths")])
        if ok:
            for x in range(len(exp["pprod"])):
                if _paths(exp, x) != _paths(got, x):
                    errs.append(f"valid_paths of pruned edge {x}: {_paths(exp, x)} != {_paths(got, x)}")
                    break
    if "diags" in parts:
        a, b = [str(s) for s in exp["diags"]], [str(s) for s in got["diags"]]
        if a != b:
            errs.append(f"diagnostics differ:\n  exp {a[:6]}\n  got {b[:6]}")
    if "blame" in parts:
        ok = all([eq("bl_stalled"), eq("bl_cause"), eq("bl_kind"), eq("bl_sub")])
        if ok:
            if [str(s) for s in exp["bl_reg"]] != [str(s) for s in got["bl_reg"]]:
                errs.append("blame registers differ")
            a, b = np.asarray(exp["bl_blame"]), np.asarray(got["bl_blame"])
            if not np.allclose(a, b, rtol=rel, atol=0.0) if rel else not np.array_equal(a, b):
                errs.append(f"blame cycles differ (max rel {np.max(np.abs(a - b) / np.maximum(np.abs(a), 1e-300)):.3g})")
            a, b = np.asarray(exp["bl_factors"]), np.asarray(got["bl_factors"])
            if not np.array_equal(np.isnan(a), np.isnan(b)):
                errs.append("blame factor presence differs")
            else:
                m = ~np.isnan(a)
                if not (np.allclose(a[m], b[m], rtol=rel, atol=0.0) if rel else np.array_equal(a[m], b[m])):
                    errs.append("blame factors differ")
    if "slice" in parts:
        eq("level")
    if "lines" in parts:
        for f in ("line_blame", "line_stall"):
            a, b = np.asarray(exp[f]), np.asarray(got[f])
            if a.shape != b.shape or not np.allclose(a, b, rtol=line_rel, atol=1e-9):
                errs.append(f"{f} differs")
    return errs


def oracle_outputs(ks, r, dialect=None) -> dict:
    """Turn an oracle.OracleResult into golden-field arrays."""
    from paper_2604_20032_b200 import diagnostics
    from paper_2604_20032_b200.diagnostics import format_ref27
    dialect = dialect or ks.dialect
    got = dict(bprod=r.prod, bcons=r.cons, bmeta=r.meta, pprod=r.p_prod, pcons=r.p_cons,
               pmeta=r.p_meta, npaths=r.p_npaths, first=r.p_first, plen=r.path_len,
               pacc=r.path_acc, level=r.level)
    got["diags"] = list(ks.prefix_diagnostics) + diagnostics.render(dialect, ks.offset, r.diags)
    got.update(blame_arrays(dialect, r.e_stalled, r.e_edge, r.e_sub, r.e_blame, r.e_factors,
                            r.p_prod, r.p_meta))
    got["line_blame"], got["line_stall"] = r.line_blame, r.line_stall
    return got


def blame_arrays(dialect, stalled, edge, sub, blame, factors, p_prod, p_meta) -> dict:
    from paper_2604_20032_b200.diagnostics import format_ref27
    edge = np.asarray(edge)
    self_ = edge < 0
    e = np.where(self_, 0, edge)
    p_prod = np.asarray(p_prod)
    p_meta = np.asarray(p_meta, dtype=np.uint32)
    meta = p_meta[e] if p_meta.size else np.zeros(edge.shape, np.uint32)
    kind = ((meta >> 27) & 7).astype(np.uint8)
    f = np.asarray(factors, dtype=np.float64).reshape(-1, 4).copy()
    f[self_] = np.nan
    reg = ["" if (s or k >= 2) else format_ref27(dialect, int(m) & 0x07FFFFFF)
           for s, k, m in zip(self_.tolist(), kind.tolist(), meta.tolist())]
    return dict(bl_stalled=np.asarray(stalled, dtype=np.int32),
                bl_cause=np.where(self_, -1, p_prod[e] if p_prod.size else -1).astype(np.int32),
                bl_kind=np.where(self_, 255, kind).astype(np.uint8),
                bl_sub=np.where(self_, np.asarray(sub), 255).astype(np.uint8),
                bl_blame=np.asarray(blame, dtype=np.float64), bl_factors=f,
                bl_reg=np.array(reg, dtype=np.str_))
