"""Canonical forms used to compare the reference, the oracle and the device.

Edges:   (producer, consumer, kind, ref|None, dep_class, ((len, accum), ...))
Blame:   (stalled, cause|None, kind|None, sub|None, blame, factors|None, register|None)
All indices are the enum positions in paper_2604_20032_b200.enums.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2604_20032_b200 import enums as E
from paper_2604_20032_b200.diagnostics import format_ref27


# ---- reference objects ----------------------------------------------------

def ref_edges(graph, with_paths=True):
    out = []
    for e in graph.edges:
        ref = None
        if e.register is not None:
            ref = (E.RC_IDX[e.register.reg_class.value], e.register.index, e.register.span)
        paths = tuple((p.length_instructions, float(p.accumulated_issue_cycles))
                      for p in e.valid_paths) if with_paths else ()
        out.append((e.producer, e.consumer, E.EK_IDX[e.kind.value], ref,
                    E.DC_IDX[e.dep_class.value], paths))
    return out


def ref_blame(entries):
    out = []
    for b in entries:
        f = None if b.factors is None else (b.factors.dist, b.factors.eff, b.factors.isu,
                                            b.factors.match)
        out.append((b.stalled, b.cause, None if b.kind is None else E.EK_IDX[b.kind.value],
                    None if b.subcategory is None else E.SB_IDX[b.subcategory.value],
                    b.blame_cycles, f, b.register))
    return out


# ---- SoA arrays -------------------------------------------------------------

def soa_edges(prod, cons, meta, npaths=None, first=None, plen=None, pacc=None):
    out = []
    prod = np.asarray(prod).tolist()
    cons = np.asarray(cons).tolist()
    meta = np.asarray(meta, dtype=np.uint32).tolist()
    if npaths is not None:
        npaths = np.asarray(npaths).tolist()
        first = np.asarray(first).tolist()
        plen = np.asarray(plen).tolist()
        pacc = np.asarray(pacc).tolist()
    for x in range(len(prod)):
        m = meta[x]
        kind = (m >> 27) & 7
        ref = None
        if kind < 2:
            ref = ((m >> 24) & 7, m & 0xFFFF, (m >> 16) & 0xFF)
        paths = ()
        if npaths is not None and npaths[x] > 0:
            f = first[x]
            paths = tuple((plen[f + q], pacc[f + q]) for q in range(npaths[x]))
        out.append((prod[x], cons[x], kind, ref, (m >> 30) & 3, paths))
    return out


def soa_blame(dialect, e_stalled, e_edge, e_sub, e_blame, e_factors, p_prod, p_meta):
    out = []
    p_prod = np.asarray(p_prod).tolist()
    p_meta = np.asarray(p_meta, dtype=np.uint32).tolist()
    for s, e, sub, bl, f in zip(np.asarray(e_stalled).tolist(), np.asarray(e_edge).tolist(),
                                np.asarray(e_sub).tolist(), np.asarray(e_blame).tolist(),
                                np.asarray(e_factors).tolist()):
        if e < 0:
            out.append((s, None, None, sub, bl, None, None))
        else:
            m = p_meta[e]
            kind = (m >> 27) & 7
            reg = format_ref27(dialect, m & 0x07FFFFFF) if kind < 2 else None
            out.append((s, p_prod[e], kind, None, bl, tuple(f), reg))
    return out


def blame_close(a, b, rel=1e-6):
    """Structural equality plus blame/factor agreement within `rel`."""
    if len(a) != len(b):
        return False, f"length {len(a)} != {len(b)}"
    for x, (u, v) in enumerate(zip(a, b)):
        if u[:4] != v[:4] or u[6] != v[6]:
            return False, f"entry {x}: {u} != {v}"
        if not math.isclose(u[4], v[4], rel_tol=rel, abs_tol=0.0):
            return False, f"entry {x}: blame {u[4]} != {v[4]}"
        if (u[5] is None) != (v[5] is None):
            return False, f"entry {x}: factors {u[5]} != {v[5]}"
        if u[5] is not None:
            for p, q in zip(u[5], v[5]):
                if not math.isclose(p, q, rel_tol=rel, abs_tol=0.0):
                    return False, f"entry {x}: factors {u[5]} != {v[5]}"
    return True, ""


def ref_slice(pruned, attached):
    """Frozen slice semantics: BFS over `pruned.incoming` from
    every instruction with S_j > 0; level = min hop count."""
    n = len(attached.cfg.instructions)
    level = [-1] * n
    frontier = []
    for j in range(n):
        if attached.stall_cycles_at(j) != 0:
            level[j] = 0
            frontier.append(j)
    lv = 0
    while frontier:
        lv += 1
        nxt = []
        for v in frontier:
            for e in pruned.incoming_edges(v):
                if level[e.producer] < 0:
                    level[e.producer] = lv
                    nxt.append(e.producer)
        frontier = nxt
    return level


def ref_lines(blame, attached, key_of):
    """Frozen per-line rollup: blame to line(cause) (self: line(stalled));
    stall to line(j).  Summed in entry / instruction order."""
    lb, ls = {}, {}
    for b in blame:
        at = b.stalled if b.cause is None else b.cause
        k = key_of(at)
        lb[k] = lb.get(k, 0.0) + b.blame_cycles
    for j in range(len(attached.cfg.instructions)):
        s = attached.stall_cycles_at(j)
        if s != 0:
            k = key_of(j)
            ls[k] = ls.get(k, 0.0) + s
    return lb, ls
