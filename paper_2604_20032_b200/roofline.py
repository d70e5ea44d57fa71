"""Algorithmic (compulsory) HBM bytes of the hot path, SURVEY.md §8(d).

Every term is counted from the actual arrays of the run: each input read
once, each output written once.  Used by bench.py for the roofline of the
dominant kernel (bytes per launch / CUDA-event launch time) and of the whole
step.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from . import abi


def _sizes(ks, wl, res):
    N, B = ks.n_instr, ks.n_blocks
    M = int(ks.opnd.shape[0])
    nu, nd = abi.unit_counts(ks)
    S = int(wl.pc.shape[0]) if wl is not None else 0
    E = int(res["bprod"].shape[0])
    Ep = int(res["pprod"].shape[0])
    P = int(res["plen"].shape[0])
    nb = int(res["e_blame"].shape[0])
    L = int(res["line_blame"].shape[0])
    cfg_edges = int(ks.succ.shape[0])
    # bytes per raw sample as the device reads them: the packed u32 stream
    # (kernels below 2^24 instructions, device.DeviceSamples default) or i32 pc + u8 cat
    SB = 4 if (N < (1 << 24) and S >= (4 << 20)) else 5
    return dict(N=N, B=B, M=M, NU=nu, ND=nd, S=S, SB=SB, E=E, Ep=Ep, P=P, NB=nb, L=L, CE=cfg_edges,
                NREG=int(res.get("n_regular", E)))


def pipeline_bytes(ks, wl, res) -> int:
    """B_alg of one step."""
    z = _sizes(ks, wl, res)
    return int(z["SB"] * z["S"] + 32 * z["N"] + 4 * (z["ND"] + z["NU"]) + 16 * z["B"] + 8 * z["CE"]
               + 24 * z["N"] + 32 * z["N"] + 16 * z["E"] + 16 * z["Ep"] + 16 * z["P"]
               + z["N"] / 8 + 4 * z["N"] + 56 * z["NB"] + 8 * z["L"])


def kernel_bytes(name: str, ks, wl, res) -> int | None:
    """Compulsory bytes of one launch of kernel `name`."""
    z = _sizes(ks, wl, res)
    N, E, Ep = z["N"], z["E"], z["Ep"]
    table = {
        # raw samples (i32 pc + u8 category) read once, class counts written once
        "bin_samples": z["SB"] * z["S"] + 32 * N,
        "bin_finalize": 32 * N + 4 * N,
        # operand CSR + offsets + block table in; per-use-event results + block summaries out
        "block_walk": 4 * z["M"] + 4 * N + 8 * N + 8 * z["B"] + 4 * z["NU"] + 8 * z["ND"],
        # candidate edges in (prod, cons, meta) + keep/npaths/pfirst/dist out + path records
        "prune_edges": 12 * E + 20 * E + 12 * z["P"] + 16 * N,
        # per-instruction sync words + CFG + raw sync keys out
        "sync_trace": 9 * N + 8 * z["B"] + 8 * z["CE"] + 8 * (E - z["NREG"]),
        # pruned incoming CSR + producers in, levels + bitmap out
        "slice": 12 * Ep + 8 * N + 4 * N + N // 8,
        # pruned edges + per-instruction profile in, per-instruction decision out
        "blame_count": 12 * Ep + 8 * Ep + 56 * N + 24 * N,
        "blame_fill": 12 * Ep + 8 * Ep + 56 * N + 56 * z["NB"],
        "link_count": 4 * z["M"] + 4 * z["NU"] + 4 * N,
        "link_fill": 4 * z["M"] + 4 * z["NU"] + 8 * z["NU"],
        "segsort_unique": 16 * z["NU"] + 4 * N,
        "lines": 16 * z["NB"] + 8 * z["L"] + 8 * N,
        # SURVEY §8(d) terms only (the unit columns are this design's own
        # derived tables, not algorithmic bytes): def / use units, the block
        # records and CFG, one query + result per use unit
        "reach_fast": 4 * (z["ND"] + z["NU"]) + 16 * z["B"] + 8 * z["CE"] + 12 * z["NU"],
        # base-graph RAW incoming of the candidates + per-candidate verdicts
        "selfblame_warp": 12 * z["E"] + 8 * N,
    }
    v = table.get(name)
    return int(v) if v is not None else None


def ncu_sectors_per_request(profiles: Path, config: str, kernel: str):
    """l1tex global-load sectors per request of `kernel` from the committed
    ncu --set full summary (profiles/ncu_kernel_stats.json)."""
    p = Path(profiles) / "ncu_kernel_stats.json"
    try:
        return json.loads(p.read_text()).get(config, {}).get(kernel, {}).get("sectors_per_request")
    except Exception:
        return None


def ncu_traffic(profiles: Path, config: str, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    from the committed ncu --set full summary (profiles/ncu_traffic.json)."""
    p = Path(profiles) / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get(config, {}).get(kernel)
    except Exception:
        return None
