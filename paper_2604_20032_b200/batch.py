"""Batch many independent kernels into one device pipeline pass.

Kernels are independent: no CFG edge, reaching-definition
search, sync chain or stage-3 path can leave a kernel — backward walks stop
at the kernel's entry block (no predecessors) and forward walks at its exit.
So the analysis of the concatenation of several kernels' instruction streams
and CFGs (block and instruction ids offset, dense unit ids recomputed over the
union) is exactly the union of the per-kernel analyses, and every per-kernel
output is a contiguous slice of the batch output:

  * raw/guard edges are consumer-sorted and sync edges producer-sorted, so a
    kernel's edges form one contiguous run in each part;
  * blame entries are ordered by stalled instruction;
  * diagnostics carry instruction indices.

Kernels are grouped by (dialect, sampling period): both are per-kernel
constants of the analysis (sync semantics, issue weights, stage 2, latency
thresholds, S_j = latency x period).  This is the segmented batching of
SURVEY.md §7.4 (config C4: 2,000 kernels) without any per-kernel launches.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .soa import KernelSoA, ProfileSoA


@dataclass
class Batch:
    kernel: KernelSoA
    profile: ProfileSoA
    pc: np.ndarray
    cat: np.ndarray
    lut: np.ndarray
    instr_off: np.ndarray        # [K+1] instruction offsets of the member kernels
    names: list

    @property
    def n_samples(self) -> int:
        return int(self.pc.shape[0])


def group_key(wl) -> tuple:
    return (wl.kernel.dialect, int(wl.profile.period))


def concat(workloads) -> Batch:
    """Concatenate workloads of one (dialect, period) group."""
    assert workloads, "empty batch"
    keys = {group_key(w) for w in workloads}
    if len(keys) != 1:
        raise ValueError(f"batch mixes dialect/period groups: {sorted(keys)}")
    dialect, period = keys.pop()
    ks_list = [w.kernel for w in workloads]
    n = np.array([k.n_instr for k in ks_list], dtype=np.int64)
    b = np.array([k.n_blocks for k in ks_list], dtype=np.int64)
    ioff = np.concatenate([[0], np.cumsum(n)])
    boff = np.concatenate([[0], np.cumsum(b)])
    # dense units over the union: per-class extent = max over kernels
    ext = np.zeros(8, dtype=np.int64)
    for k in ks_list:
        op = np.asarray(k.opnd, dtype=np.uint32)
        if op.size:
            rc = (op >> 24) & 7
            top = (op & 0xFFFF) + ((op >> 16) & 0xFF)
            for c in np.unique(rc):
                ext[c] = max(ext[c], int(top[rc == c].max()))
    unit_base = np.concatenate([[0], np.cumsum(ext)[:-1]]).astype(np.int32)
    opnd = np.concatenate([k.opnd for k in ks_list]).astype(np.uint32)
    opnd_counts = np.concatenate([np.diff(k.opnd_ptr) for k in ks_list])
    opnd_ptr = np.concatenate([[0], np.cumsum(opnd_counts)]).astype(np.int32)

    def cat_shift(name, shift):
        return np.concatenate([np.asarray(getattr(k, name), dtype=np.int64) + s
                               for k, s in zip(ks_list, shift)]).astype(np.int32)

    succ_counts = np.concatenate([np.diff(k.succ_ptr) for k in ks_list])
    pred_counts = np.concatenate([np.diff(k.pred_ptr) for k in ks_list])
    lines = ks_list[0].lines
    kernel = KernelSoA(
        name=f"batch[{dialect},{period}]x{len(ks_list)}", dialect=dialect,
        opclass=np.concatenate([k.opclass for k in ks_list]),
        block_of=cat_shift("block_of", boff[:-1]),
        opnd_ptr=opnd_ptr, opnd=opnd,
        sync_kind=np.concatenate([k.sync_kind for k in ks_list]),
        sync_a=np.concatenate([k.sync_a for k in ks_list]),
        sync_b=np.concatenate([k.sync_b for k in ks_list]),
        blk_first=cat_shift("blk_first", ioff[:-1]), blk_last=cat_shift("blk_last", ioff[:-1]),
        succ_ptr=np.concatenate([[0], np.cumsum(succ_counts)]).astype(np.int32),
        succ=cat_shift("succ", boff[:-1]),
        pred_ptr=np.concatenate([[0], np.cumsum(pred_counts)]).astype(np.int32),
        pred=cat_shift("pred", boff[:-1]),
        unit_base=unit_base, n_units=int(ext.sum()),
        offset=np.concatenate([k.offset for k in ks_list]),
        line_id=np.concatenate([k.line_id for k in ks_list]).astype(np.int32),
        lines=lines, seg_block=boff.astype(np.int32))
    ps = [w.profile for w in workloads]
    profile = ProfileSoA(
        period=period, lat=np.concatenate([p.lat for p in ps]),
        cls_cnt=np.concatenate([np.asarray(p.cls_cnt).reshape(-1, 8) for p in ps]),
        exec_cnt=np.concatenate([p.exec_cnt for p in ps]),
        total=np.concatenate([p.total for p in ps]),
        eff=np.concatenate([p.eff for p in ps]),
        sampled=np.concatenate([p.sampled for p in ps]))
    pc = np.concatenate([np.asarray(w.pc, dtype=np.int64) + o
                         for w, o in zip(workloads, ioff[:-1])]).astype(np.int32)
    cat = np.concatenate([w.cat for w in workloads])
    luts = {w.lut.tobytes() for w in workloads}
    assert len(luts) == 1
    return Batch(kernel=kernel, profile=profile, pc=pc, cat=cat, lut=workloads[0].lut,
                 instr_off=ioff, names=[k.name for k in ks_list])


def split_result(batch: Batch, r: dict) -> list[dict]:
    """Per-kernel slices of a batch result (indices re-based to the kernel)."""
    out = []
    io = batch.instr_off
    nreg, preg = r["n_regular"], r["p_n_regular"]
    for x in range(len(batch.names)):
        lo, hi = int(io[x]), int(io[x + 1])
        d = {}
        # base edges: regular part by consumer, sync part by producer
        bc, bp = r["bcons"], r["bprod"]
        sel_r = np.flatnonzero((bc[:nreg] >= lo) & (bc[:nreg] < hi))
        sel_s = nreg + np.flatnonzero((bp[nreg:] >= lo) & (bp[nreg:] < hi))
        sel = np.concatenate([sel_r, sel_s])
        d["bprod"], d["bcons"], d["bmeta"] = bp[sel] - lo, bc[sel] - lo, r["bmeta"][sel]
        pc_, pp = r["pcons"], r["pprod"]
        selr = np.flatnonzero((pc_[:preg] >= lo) & (pc_[:preg] < hi))
        sels = preg + np.flatnonzero((pp[preg:] >= lo) & (pp[preg:] < hi))
        psel = np.concatenate([selr, sels])
        remap = np.full(pp.shape[0], -1, dtype=np.int64)
        remap[psel] = np.arange(psel.shape[0])
        d["pprod"], d["pcons"], d["pmeta"] = pp[psel] - lo, pc_[psel] - lo, r["pmeta"][psel]
        d["npaths"], d["first"] = r["npaths"][psel], r["first"][psel]
        d["plen"], d["pacc"] = r["plen"], r["pacc"]
        es = r["e_stalled"]
        esel = np.flatnonzero((es >= lo) & (es < hi))
        d["e_stalled"] = es[esel] - lo
        d["e_edge"] = np.where(r["e_edge"][esel] < 0, -1, remap[np.maximum(r["e_edge"][esel], 0)])
        d["e_sub"], d["e_blame"] = r["e_sub"][esel], r["e_blame"][esel]
        d["e_factors"] = r["e_factors"][esel]
        d["level"] = r["level"][lo:hi]
        dr = r["diag_records"]
        ds = dr[(dr[:, 1] >= lo) & (dr[:, 1] < hi)].copy() if dr.size else dr
        if ds.size:
            ds[:, 1] -= lo
            cap = ds[:, 0] == 4          # path-capped: a0 = consumer index
            ds[cap, 2] -= lo
        d["diag_records"] = ds
        out.append(d)
    return out
