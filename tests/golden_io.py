"""Golden-vector fixture format (no dependency on the reference package).

A fixture file is one compressed npz holding many cases; case `i` stores its
arrays under keys `"{i}/<field>"`.  Each case = one kernel SoA + profile SoA +
analysis config + the outputs the *reference* produced for them:

  base edges   bprod/bcons/bmeta                (build_graph, depgraph.py:507)
  pruned       pprod/pcons/pmeta + npaths/first/plen/pacc   (run_pruning)
  diagnostics  diags (str)                      (DependencyGraph.diagnostics)
  blame        bl_stalled/bl_cause/bl_kind/bl_sub/bl_blame/bl_factors/bl_reg
  slice        level                            (frozen slice semantics)
  lines        line_blame/line_stall over the case's line table
"""

from __future__ import annotations

import json

import numpy as np

from paper_2604_20032_b200.soa import KernelSoA, ProfileSoA

K_FIELDS = ("opclass", "block_of", "opnd_ptr", "opnd", "sync_kind", "sync_a", "sync_b",
            "blk_first", "blk_last", "succ_ptr", "succ", "pred_ptr", "pred", "unit_base",
            "offset", "line_id")
P_FIELDS = ("lat", "cls_cnt", "exec_cnt", "total", "eff", "sampled")


def pack_case(ks: KernelSoA, pf: ProfileSoA, cfg: dict, expected: dict) -> dict:
    d = {f"k_{f}": getattr(ks, f) for f in K_FIELDS}
    d.update({f"p_{f}": getattr(pf, f) for f in P_FIELDS})
    meta = dict(name=ks.name, dialect=ks.dialect, n_units=ks.n_units, lines=list(ks.lines),
                prefix=list(ks.prefix_diagnostics), period=pf.period, cfg=cfg)
    d["meta"] = np.array(json.dumps(meta))
    for k, v in expected.items():
        d[f"x_{k}"] = v
    return d


def save(path, cases: list[dict]):
    """Concatenate every field across cases (one npz member per field plus a
    per-case length vector) to keep the archive small."""
    fields = sorted({k for c in cases for k in c if k != "meta"})
    flat = {"metas": np.array([str(c["meta"]) for c in cases])}
    for f in fields:
        parts = [np.asarray(c[f]) for c in cases]
        flat[f"len/{f}"] = np.array([p.shape[0] if p.ndim else 1 for p in parts], dtype=np.int64)
        flat[f"cat/{f}"] = np.concatenate([p.reshape(-1, *p.shape[1:]) if p.ndim else p.reshape(1)
                                           for p in parts])
    np.savez_compressed(path, **flat)


def load(path):
    z = np.load(path, allow_pickle=False)
    metas = z["metas"]
    n = metas.shape[0]
    groups = [{"meta": metas[i]} for i in range(n)]
    for key in z.files:
        if not key.startswith("cat/"):
            continue
        f = key[4:]
        lens = z[f"len/{f}"]
        data = z[key]
        off = np.concatenate([[0], np.cumsum(lens)])
        for i in range(n):
            groups[i][f] = data[off[i]:off[i + 1]]
    out = []
    for g in groups:
        meta = json.loads(str(g["meta"]))
        ks = KernelSoA(name=meta["name"], dialect=meta["dialect"], n_units=meta["n_units"],
                       lines=meta["lines"], prefix_diagnostics=tuple(meta["prefix"]),
                       **{f: g[f"k_{f}"] for f in K_FIELDS})
        pf = ProfileSoA(period=meta["period"], **{f: g[f"p_{f}"] for f in P_FIELDS})
        exp = {k[2:]: v for k, v in g.items() if k.startswith("x_")}
        out.append((ks, pf, meta["cfg"], exp))
    return out


def config_of(cfg: dict, dialect: str):
    from paper_2604_20032_b200 import abi
    return abi.make_config(cfg["stage_mask"], cfg["prune_exec"], cfg["max_paths"],
                           cfg["max_depth"], cfg.get("thresholds"), dialect)
