"""Render typed diagnostic records into the reference's exact strings.

The device emits (code, instr, a0, a1, a2, seq) records in any order; this
module orders them the way the reference appends them and formats them with
the reference's f-strings:

  unresolved use   depgraph.py:219-222   (per instruction, operand order, dedup (i, name))
  waitcnt exceeds  depgraph.py:395-399   (per wait, vmcnt before lgkmcnt)
  no setter        depgraph.py:461-462, 480-481 (per wait, ascending id)
  path capped      analysis.py:277-284   (edge-list order)
"""

from __future__ import annotations

import numpy as np

from . import enums as E

_GROUP = {1: 0, 2: 1, 3: 1, 4: 2}


def format_register(dialect: str, rc: int, index: int, span: int) -> str:
    """isa.py:320-336"""
    cls = E.REG_CLASSES[rc]
    if cls == "predicate":
        return f"P{index}"
    if cls == "barrier":
        return f"B{index}"
    if dialect == "amd":
        base = "v" if cls == "vector_gpr" else "s"
        return f"{base}{index}" if span == 1 else f"{base}[{index}:{index + span - 1}]"
    if dialect == "intel":
        return f"r{index}" if span == 1 else f"r{index}:+{span - 1}"
    prefix = "UR" if cls == "uniform" else "R"
    return f"{prefix}{index}" if span == 1 else f"{prefix}{index}:+{span - 1}"


def format_ref27(dialect: str, ref27: int) -> str:
    return format_register(dialect, (ref27 >> 24) & 7, ref27 & 0xFFFF, (ref27 >> 16) & 0xFF)


def order(records: np.ndarray) -> np.ndarray:
    """Sort device diagnostic records into reference emission order."""
    records = np.asarray(records, dtype=np.int32).reshape(-1, 6)
    if records.shape[0] == 0:
        return records
    group = np.array([_GROUP[int(c)] for c in records[:, 0]], dtype=np.int64)
    instr = records[:, 1].astype(np.int64)
    seq = records[:, 5].astype(np.int64)
    # path-capped records are ordered by edge index alone
    instr = np.where(group == 2, 0, instr)
    idx = np.lexsort((seq, instr, group))
    return records[idx]


def render(dialect: str, offsets, records, ordered: bool = False) -> list[str]:
    recs = records if ordered else order(records)
    out: list[str] = []
    seen_unresolved = set()
    for code, instr, a0, a1, a2, _seq in np.asarray(recs).tolist():
        if code == 1:
            name = format_ref27(dialect, a0 & 0x07FFFFFF)
            key = (instr, name)
            if key in seen_unresolved:
                continue
            seen_unresolved.add(key)
            out.append(f"use of undefined register {name} at 0x{int(offsets[instr]):x} (no edge)")
        elif code == 2:
            counter = "vmcnt" if a0 == 0 else "lgkmcnt"
            out.append(f"waitcnt at 0x{int(offsets[instr]):x}: {counter}({a1}) exceeds {a2} pending "
                       f"operation(s); listing may be truncated")
        elif code == 3:
            if dialect == "nvidia":
                out.append(f"wait on B{a0} at 0x{int(offsets[instr]):x} has no reachable setter")
            else:
                out.append(f"wait on sbid {a0} at 0x{int(offsets[instr]):x} has no reachable setter")
        elif code == 4:
            tail = "kept with partial paths" if a1 == 1 else "conservatively kept"
            out.append(f"path enumeration capped for edge 0x{int(offsets[instr]):x}"
                       f" -> 0x{int(offsets[a0]):x}; {tail}")
        else:
            raise ValueError(f"unknown diagnostic code {code}")
    return out
