"""SoA-level device ops: one function per C-ABI entry point outside the fused
pipeline (include/leo_b200.h), arrays in and arrays out.

api.py converts the reference's objects to and from these arrays; the GPU
parity tests call these functions directly on the golden vectors.  Every
variable-size output uses the library's capacity + device counter protocol:
the call is repeated with larger buffers when the device reports an
overflow.  No computation happens here (no CPU fallback).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import abi, device, diagnostics
from ._lib import check, lib


def _stream(dev):
    return torch.cuda.current_stream(dev).cuda_stream


def _i32(n, dev):
    return torch.zeros(max(int(n), 1), dtype=torch.int32, device=dev)


def _f64(n, dev):
    return torch.zeros(max(int(n), 1), dtype=torch.float64, device=dev)


def up(a, dev, dtype=np.int32):
    return device.to_device(np.ascontiguousarray(np.asarray(a, dtype=dtype)), dev)


class DevEdges:
    """An edge list (+ valid_paths) in HBM.  canonical: library-made (raw/guard
    edges consumer-sorted first, n_regular valid); else arbitrary order
    (LeoEdges.n_regular = NULL)."""

    def __init__(self, dev, prod, cons, meta, count, canonical, n_regular=None,
                 first=None, npaths=None, plen=None, pacc=None, pcount=0):
        self.dev = dev
        self.prod, self.cons, self.meta = prod, cons, meta
        self.count = int(count)
        self.canonical = canonical
        self.ctr = torch.tensor([self.count, n_regular or 0, pcount or 0, 0], dtype=torch.int32, device=dev)
        self.first, self.npaths, self.plen, self.pacc = first, npaths, plen, pacc
        self.pcount = int(pcount or 0)

    @classmethod
    def from_arrays(cls, dev, prod, cons, meta, npaths=None, first=None, plen=None, pacc=None,
                    canonical=False, n_regular=None):
        n = len(prod)
        t = dict(prod=up(prod, dev), cons=up(cons, dev),
                 meta=up(np.asarray(meta, np.uint32).view(np.int32), dev))
        if npaths is not None and n and len(plen):
            t.update(npaths=up(npaths, dev), first=up(first, dev), plen=up(plen, dev),
                     pacc=up(pacc, dev, np.float64), pcount=len(plen))
        return cls(dev, count=n, canonical=canonical, n_regular=n_regular, **t)

    def edges_struct(self):
        cp = self.ctr.data_ptr()
        return abi.LeoEdges(max(self.count, 1), self.prod.data_ptr(), self.cons.data_ptr(),
                            self.meta.data_ptr(), cp, cp + 4 if self.canonical else None)

    def paths_struct(self):
        if self.first is None:
            return None
        return abi.LeoPaths(max(self.pcount, 1), self.first.data_ptr(), self.npaths.data_ptr(), None,
                            self.plen.data_ptr(), self.pacc.data_ptr(), self.ctr.data_ptr() + 8)


def _byref(s):
    return C.byref(s) if s is not None else None


def build(dk: device.DeviceKernel) -> dict:
    """leo_build_graph: base edges (canonical) + ordered diagnostic records."""
    dev, ks = dk.device, dk.ks
    n = ks.n_instr
    nu, _ = abi.unit_counts(ks)
    cap, dcap = 3 * nu + 2 * n + 1024, 2 * n + 1024
    for _ in range(6):
        ctr = _i32(4, dev)
        prod, cons, meta = _i32(cap, dev), _i32(cap, dev), _i32(cap, dev)
        drec = _i32(6 * dcap, dev)
        cp = ctr.data_ptr()
        e = abi.LeoEdges(cap, prod.data_ptr(), cons.data_ptr(), meta.data_ptr(), cp, cp + 4)
        dg = abi.LeoDiags(dcap, drec.data_ptr(), cp + 8)
        check(lib().leo_build_graph(C.byref(dk.struct), None, C.byref(e), C.byref(dg), cp + 12,
                                    _stream(dev)), "leo_build_graph")
        c = ctr.cpu().numpy()
        st = int(np.uint32(c[3]))
        if st & abi.ST_BAD_INPUT:
            raise ValueError("device reported malformed input (a block with more than two successors)")
        if c[0] <= cap and c[2] <= dcap and not st:
            break
        cap, dcap = max(cap, int(c[0])) * 2 + 1024, max(dcap, int(c[2])) * 2 + 1024
    else:
        raise RuntimeError("leo_build_graph: buffers kept overflowing")
    m, nreg = int(c[0]), int(c[1])
    return dict(bprod=prod[:m].cpu().numpy(), bcons=cons[:m].cpu().numpy(),
                bmeta=meta[:m].cpu().numpy().view(np.uint32), n_regular=nreg,
                diag_records=diagnostics.order(drec[:6 * int(c[2])].cpu().numpy().reshape(-1, 6)),
                edges=DevEdges(dev, prod, cons, meta, m, True, nreg))


def reach_in(dk: device.DeviceKernel):
    """leo_reaching_definitions: (set_off[B*U+1], defs) over (block, unit) pairs
    (set semantics: a def may be listed twice in a set, when the search reached
    two blocks of one fallthrough run that share their nearest definition)."""
    dev, ks = dk.device, dk.ks
    B, U = ks.n_blocks, ks.n_units
    cap = 4 * B * U + 1024
    for _ in range(6):
        ctr = _i32(4, dev)
        off, defs = _i32(B * U + 1, dev), _i32(cap, dev)
        out = abi.LeoReachIn(cap, off.data_ptr(), defs.data_ptr(), ctr.data_ptr())
        caps = abi.LeoCaps()
        caps.query_results = cap
        check(lib().leo_reaching_definitions(C.byref(dk.struct), C.byref(caps), C.byref(out),
                                             ctr.data_ptr() + 4, _stream(dev)), "leo_reaching_definitions")
        c = ctr.cpu().numpy()
        if not (int(np.uint32(c[1])) & abi.ST_SCRATCH_OVERFLOW) and c[0] <= cap:
            break
        cap = max(cap, int(c[0])) * 2 + 1024
    else:
        raise RuntimeError("leo_reaching_definitions: buffers kept overflowing")
    return off[:B * U + 1].cpu().numpy(), defs[:int(c[0])].cpu().numpy()


def liveness_filter(dk: device.DeviceKernel, prod, cons, meta) -> np.ndarray:
    """leo_liveness_filter: keep[e] for links (prod, cons, ref27 | kind << 27)."""
    dev = dk.device
    n = len(prod)
    if n == 0:
        return np.zeros(0, np.uint8)
    d = DevEdges.from_arrays(dev, prod, cons, meta)
    keep = torch.zeros(n, dtype=torch.uint8, device=dev)
    check(lib().leo_liveness_filter(C.byref(dk.struct), C.byref(d.edges_struct()), keep.data_ptr(),
                                    _stream(dev)), "leo_liveness_filter")
    return keep.cpu().numpy()


def prune(dk: device.DeviceKernel, dp: device.DeviceProfile, cfg: abi.LeoConfig, d: DevEdges):
    """leo_prune over any edge list (input valid_paths carried): (result arrays,
    DevEdges of the pruned list)."""
    dev = dk.device
    n = d.count
    pcap = max(2 * n, 64) + d.pcount
    dcap = n + 64
    for _ in range(6):
        ctr = _i32(8, dev)
        prod, cons, meta = _i32(n, dev), _i32(n, dev), _i32(n, dev)
        first, npaths = _i32(n, dev), _i32(n, dev)
        dist = _f64(n, dev)
        plen, pacc = _i32(pcap, dev), _f64(pcap, dev)
        drec = _i32(6 * dcap, dev)
        cp = ctr.data_ptr()
        out = abi.LeoEdges(max(n, 1), prod.data_ptr(), cons.data_ptr(), meta.data_ptr(), cp, cp + 4)
        paths = abi.LeoPaths(pcap, first.data_ptr(), npaths.data_ptr(), dist.data_ptr(),
                             plen.data_ptr(), pacc.data_ptr(), cp + 8)
        dg = abi.LeoDiags(dcap, drec.data_ptr(), cp + 12)
        check(lib().leo_prune(C.byref(dk.struct), C.byref(dp.struct), C.byref(cfg), C.byref(d.edges_struct()),
                              _byref(d.paths_struct()), C.byref(out), C.byref(paths), C.byref(dg), cp + 16,
                              _stream(dev)), "leo_prune")
        c = ctr.cpu().numpy()
        st = int(np.uint32(c[4]))
        if st & abi.ST_BAD_INPUT:
            raise ValueError("device reported malformed input (a block with more than two successors)")
        if st & abi.ST_SCRATCH_OVERFLOW:
            raise RuntimeError("leo_prune: slow-path list overflowed")
        if st & abi.ST_PATH_OVERFLOW or c[2] > pcap:
            pcap = max(pcap, int(c[2])) * 2 + 1024
            continue
        if st & abi.ST_DIAG_OVERFLOW or c[3] > dcap:
            dcap = max(dcap, int(c[3])) * 2 + 64
            continue
        break
    else:
        raise RuntimeError("leo_prune: buffers kept overflowing")
    m, npa = int(c[0]), int(c[2])
    h = lambda t, q: t[:q].cpu().numpy()  # noqa: E731
    r = dict(pprod=h(prod, m), pcons=h(cons, m), pmeta=h(meta, m).view(np.uint32), npaths=h(npaths, m),
             first=h(first, m), plen=h(plen, npa), pacc=h(pacc, npa),
             diag_records=diagnostics.order(h(drec, 6 * int(c[3])).reshape(-1, 6)))
    has = npa > 0 and bool((r["npaths"] > 0).any())
    out_d = DevEdges(dev, prod, cons, meta, m, False, first=first if has else None,
                     npaths=npaths if has else None, plen=plen if has else None,
                     pacc=pacc if has else None, pcount=npa)
    return r, out_d


def blame(dk, dp, d: DevEdges, base: DevEdges | None = None, lines: bool = False) -> dict:
    """leo_blame over any edge list: entries (+ per-line vectors)."""
    dev = dk.device
    n = dk.ks.n_instr
    cap = d.count + n + 1024
    nl = dk.n_lines
    lb, ls = _f64(nl, dev), _f64(nl, dev)
    for _ in range(4):
        ctr = _i32(4, dev)
        st_, ed = _i32(cap, dev), _i32(cap, dev)
        sub = torch.empty(max(cap, 1), dtype=torch.uint8, device=dev)
        bl, fa = _f64(cap, dev), _f64(4 * cap, dev)
        out = abi.LeoBlame(cap, st_.data_ptr(), ed.data_ptr(), sub.data_ptr(), bl.data_ptr(),
                           fa.data_ptr(), ctr.data_ptr())
        check(lib().leo_blame(C.byref(dk.struct), C.byref(dp.struct), C.byref(d.edges_struct()),
                              _byref(d.paths_struct()), _byref(base.edges_struct() if base else None),
                              dk.line_id.data_ptr() if lines else None, nl if lines else 0, C.byref(out),
                              lb.data_ptr() if lines else None, ls.data_ptr() if lines else None,
                              ctr.data_ptr() + 4, _stream(dev)), "leo_blame")
        c = ctr.cpu().numpy()
        if not (int(np.uint32(c[1])) & (abi.ST_BLAME_OVERFLOW | abi.ST_SCRATCH_OVERFLOW)) and c[0] <= cap:
            break
        cap = max(cap, int(c[0])) * 2 + 1024
    else:
        raise RuntimeError("leo_blame: buffers kept overflowing")
    m = int(c[0])
    h = lambda t, q: t[:q].cpu().numpy()  # noqa: E731
    return dict(e_stalled=h(st_, m), e_edge=h(ed, m), e_sub=h(sub, m), e_blame=h(bl, m),
                e_factors=h(fa, 4 * m).reshape(-1, 4), line_blame=h(lb, nl), line_stall=h(ls, nl))


def self_blame(dk, dp, base: DevEdges | None, index):
    """leo_self_blame: (SelfBlame index, S_j) per given instruction."""
    dev = dk.device
    index = np.asarray(index, dtype=np.int32)
    n = len(index)
    sub = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
    cyc = _f64(n, dev)
    idx = up(index, dev)              # (kept alive until the results are read back)
    check(lib().leo_self_blame(C.byref(dk.struct), C.byref(dp.struct),
                               _byref(base.edges_struct() if base else None), n, idx.data_ptr(),
                               sub.data_ptr(), cyc.data_ptr(), _stream(dev)), "leo_self_blame")
    return sub[:n].cpu().numpy(), cyc[:n].cpu().numpy()


def slice_levels(dk, dp, d: DevEdges) -> np.ndarray:
    """leo_slice: hop level per instruction (-1 outside the slice)."""
    dev = dk.device
    n = dk.ks.n_instr
    level, bitmap = _i32(n, dev), _i32((n + 31) // 32, dev)
    check(lib().leo_slice(C.byref(dk.struct), C.byref(dp.struct), C.byref(d.edges_struct()),
                          bitmap.data_ptr(), level.data_ptr(), _stream(dev)), "leo_slice")
    return level[:n].cpu().numpy()


def coverage(dk, d: DevEdges):
    """leo_coverage: (nodes with incoming edges, qualifying nodes)."""
    out = _i32(2, dk.device)
    check(lib().leo_coverage(C.byref(dk.struct), C.byref(d.edges_struct()), out.data_ptr(),
                             _stream(dk.device)), "leo_coverage")
    nodes, qual = out.cpu().numpy().tolist()
    return nodes, qual


def rank_hotspots(dk, dp, top_n: int, include_unsampled: bool) -> list:
    hot, nh = _i32(top_n, dk.device), _i32(1, dk.device)
    check(lib().leo_rank_hotspots(C.byref(dk.struct), C.byref(dp.struct), int(top_n),
                                  1 if include_unsampled else 0, hot.data_ptr(), nh.data_ptr(),
                                  _stream(dk.device)), "leo_rank_hotspots")
    return hot[:int(nh.item())].cpu().numpy().tolist()


def trace_chain(dk, stalled, cause, blame_cycles, start: int, max_depth: int):
    """leo_trace_chain: (hop instructions, entry index per hop, self entry)."""
    dev = dk.device
    node, ent, ln, sf = _i32(max_depth, dev), _i32(max_depth, dev), _i32(1, dev), _i32(1, dev)
    # the uploads stay referenced until the results are read back (the call is asynchronous)
    d_st, d_ca, d_bl = up(stalled, dev), up(cause, dev), up(blame_cycles, dev, np.float64)
    check(lib().leo_trace_chain(C.byref(dk.struct), len(stalled), d_st.data_ptr(), d_ca.data_ptr(),
                                d_bl.data_ptr(), int(start), int(max_depth), node.data_ptr(), ent.data_ptr(),
                                ln.data_ptr(), sf.data_ptr(), _stream(dev)), "leo_trace_chain")
    n = int(ln.item())
    return node[:n].cpu().numpy().tolist(), ent[:n].cpu().numpy().tolist(), int(sf.item())


def line_rollup(dk, dp, stalled, cause, blame_cycles):
    """leo_line_rollup of any blame-entry list: (line_blame, line_stall)."""
    dev = dk.device
    nl = dk.n_lines
    lb, ls = _f64(nl, dev), _f64(nl, dev)
    d_st, d_ca, d_bl = up(stalled, dev), up(cause, dev), up(blame_cycles, dev, np.float64)
    check(lib().leo_line_rollup(C.byref(dk.struct), C.byref(dp.struct), len(stalled), d_st.data_ptr(),
                                d_ca.data_ptr(), d_bl.data_ptr(), dk.line_id.data_ptr(), nl, lb.data_ptr(),
                                ls.data_ptr(), _stream(dev)), "leo_line_rollup")
    return lb[:nl].cpu().numpy(), ls[:nl].cpu().numpy()
