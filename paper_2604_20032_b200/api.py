"""Public API: the reference analyzer's names and types, backed by the CUDA path.

Drop-in for the stalltrace hot path (`stalltrace/__init__.py:9-64`); every
function takes and returns the reference's own objects and computes on the
GPU through libleo_b200.so (no CPU fallback):

    build_graph(attached) -> DependencyGraph                  depgraph.py:507   leo_build_graph
    reaching_definitions(cfg) -> [ {unit: frozenset} ]        depgraph.py:135   leo_reaching_definitions
    per_use_link(cfg, reach_in) -> (links, diags)             depgraph.py:188   leo_build_graph (raw/guard)
    liveness_filter(cfg, links) -> links                      depgraph.py:274   leo_liveness_filter
    trace_waitcnt / trace_barriers / trace_swsb(cfg)          depgraph.py:402-482  leo_build_graph (sync)
    dump_graph(graph) -> str                                  depgraph.py:531   (host formatting)
    run_pruning(graph, config) -> DependencyGraph             analysis.py:302   leo_prune
    prune_opcode / prune_barrier / prune_latency / prune_execution  analysis.py:143-299  leo_prune
    attribute_blame(graph, base_graph=None) -> [BlameEntry]   analysis.py:431   leo_blame
    self_blame(index, attached, base_graph=None) -> BlameEntry analysis.py:414  leo_self_blame
    trace_chain(graph, blame, start, max_depth=32)            analysis.py:499   leo_trace_chain
    single_dep_coverage(graph) -> Coverage                    analysis.py:547   leo_coverage
    rank_hotspots(attached, top_n, include_unsampled=False)   report.py:96      leo_rank_hotspots

plus the two hot-path products the reference does not have:

    backward_slice(graph) -> (frozenset[int], dict[int, int])  leo_slice
    line_blame(graph, blame=None) -> (dict[str, float], dict[str, float])  leo_line_rollup

a fused `analyze`, and `Session`, the SoA-level entry a profiling service
uses (raw PC-sample stream in, blame entries + per-line totals out).

Graphs may be ANY DependencyGraph (the reference's tests chain stages and
build graphs by hand): a graph this module produced keeps its device edge
list; any other graph's edges are marshalled to the device in list order
(LeoEdges.n_regular = NULL: arbitrary order, include/leo_b200.h).  Outputs
are built from `stalltrace` classes when the inputs are stalltrace objects,
else from the same-named mirrors in `paper_2604_20032_b200.types`.
"""

from __future__ import annotations

import ctypes as C
import os
import dataclasses
import weakref

import numpy as np
import torch

from . import _lib, abi, device, diagnostics, ops, report, soa, types
from . import enums as E

_DEVICE = None


def _dev():
    global _DEVICE
    if _DEVICE is None:
        if not torch.cuda.is_available():
            raise RuntimeError("the LEO B200 analysis path needs a CUDA device (no CPU fallback)")
        _DEVICE = torch.device("cuda", torch.cuda.current_device())
    return _DEVICE


def _ns(obj):
    """Output type namespace matching the input objects' package."""
    mod = type(obj).__module__
    if mod.startswith("stalltrace"):
        import stalltrace.analysis as an
        import stalltrace.depgraph as dg
        import stalltrace.isa as isa
        return types.Namespace.from_modules(dg, an, isa)
    return types.Namespace.mirror()


# --------------------------------------------------------------------------
# per-object device state, keyed by identity (frozen reference dataclasses
# hash by value: hashing a whole KernelCfg per lookup would cost O(N))

class _IdCache:
    def __init__(self):
        self.d = {}

    def get(self, obj):
        hit = self.d.get(id(obj))
        if hit is not None and hit[0]() is obj:
            return hit[1]
        return None

    def put(self, obj, val):
        key = id(obj)
        try:
            ref = weakref.ref(obj, lambda _r, k=key: self.d.pop(k, None))
        except TypeError:
            return val
        self.d[key] = (ref, val)
        return val


class _Kern:
    """A kernel (cfg or attached kernel) as device SoA."""

    def __init__(self, ks, prof):
        self.ks, self.prof = ks, prof
        self.dk = device.DeviceKernel(ks, _dev())
        self.dp = device.DeviceProfile(prof, ks.n_instr, _dev())


_kernels = _IdCache()
_graphs = _IdCache()


def _zero_profile(n):
    return soa.ProfileSoA(period=1, lat=np.zeros(n, np.int32), cls_cnt=np.zeros((n, 8), np.int32),
                          exec_cnt=np.full(n, -1, np.int64), total=np.full(n, -1, np.int32),
                          eff=np.ones(n, np.float64), sampled=np.zeros(n, np.uint8))


def _kern(obj) -> _Kern:
    """Device SoA of an AttachedKernel (cfg + profile) or a bare KernelCfg."""
    k = _kernels.get(obj)
    if k is None:
        if hasattr(obj, "cfg") and hasattr(obj, "samples"):
            ks, prof = soa.encode_attached(obj)
        else:
            ks = soa.encode_cfg(obj)
            prof = _zero_profile(ks.n_instr)
        k = _kernels.put(obj, _Kern(ks, prof))
    return k


def _ref27(r):
    return r.index | (r.span << 16) | (E.RC_IDX[r.reg_class.value] << 24)


def _marshal(graph) -> ops.DevEdges:
    """A DependencyGraph's edges, in list order, to the device (arbitrary order)."""
    edges = graph.edges
    n = len(edges)
    prod = np.empty(n, np.int32)
    cons = np.empty(n, np.int32)
    meta = np.empty(n, np.uint32)
    npaths = np.zeros(n, np.int32)
    first = np.full(n, -1, np.int32)
    plen, pacc = [], []
    for x, e in enumerate(edges):
        prod[x], cons[x] = e.producer, e.consumer
        r27 = 0 if e.register is None else _ref27(e.register)
        meta[x] = r27 | (E.EK_IDX[e.kind.value] << 27) | (E.DC_IDX[e.dep_class.value] << 30)
        if e.valid_paths:
            first[x] = len(plen)
            npaths[x] = len(e.valid_paths)
            for pr in e.valid_paths:
                plen.append(pr.length_instructions)
                pacc.append(pr.accumulated_issue_cycles)
    return ops.DevEdges.from_arrays(_dev(), prod, cons, meta, npaths, first, np.asarray(plen, np.int32),
                                    np.asarray(pacc, np.float64))


def _dev_edges(graph) -> ops.DevEdges:
    d = _graphs.get(graph)
    if d is None:
        d = _graphs.put(graph, _marshal(graph))
    return d


# --------------------------------------------------------------------------
# device results -> reference objects

def _edges(ns, ks, prod, cons, meta, npaths=None, first=None, plen=None, pacc=None):
    out = []
    rcs = [ns.RegClass(v) for v in E.REG_CLASSES]
    kinds = [ns.EdgeKind(v) for v in E.EDGE_KINDS]
    dcs = [ns.DepClass(v) for v in E.DEP_CLASSES]
    prod, cons, meta = prod.tolist(), cons.tolist(), np.asarray(meta).astype(np.uint32).tolist()
    if npaths is not None:
        npaths, first, plen, pacc = npaths.tolist(), first.tolist(), plen.tolist(), pacc.tolist()
    refs = {}
    for x in range(len(prod)):
        m = meta[x]
        kind = (m >> 27) & 7
        reg = None
        if kind < 2:
            r27 = m & 0x07FFFFFF
            reg = refs.get(r27)
            if reg is None:
                reg = refs[r27] = ns.RegisterRef(rcs[(m >> 24) & 7], m & 0xFFFF, (m >> 16) & 0xFF)
        paths = ()
        if npaths is not None and npaths[x] > 0:
            f = first[x]
            paths = tuple(ns.PathRecord(plen[f + q], pacc[f + q]) for q in range(npaths[x]))
        out.append(ns.DepEdge(producer=prod[x], consumer=cons[x], kind=kinds[kind], register=reg,
                              dep_class=dcs[(m >> 30) & 3], valid_paths=paths))
    return tuple(out)


def _split_diags(ks, r):
    recs = diagnostics.order(r["diag_records"])
    build = recs[recs[:, 0] != abi.DIAG_PATH_CAPPED] if recs.size else recs
    prune = recs[recs[:, 0] == abi.DIAG_PATH_CAPPED] if recs.size else recs
    return (diagnostics.render(ks.dialect, ks.offset, build, ordered=True),
            diagnostics.render(ks.dialect, ks.offset, prune, ordered=True))


def _config_of(config, dialect):
    if config is None:
        return abi.make_config(dialect=dialect)
    if isinstance(config, abi.LeoConfig):
        return config
    return abi.config_from_reference(config, dialect)


# --------------------------------------------------------------------------
# build_graph and its sub-steps (depgraph.py)

def _build(k: _Kern) -> dict:
    b = ops.build(k.dk)
    recs = b["diag_records"]
    b["unresolved"] = diagnostics.render(k.ks.dialect, k.ks.offset, recs[recs[:, 0] == abi.DIAG_UNRESOLVED],
                                         ordered=True)
    b["sync_diags"] = diagnostics.render(k.ks.dialect, k.ks.offset, recs[recs[:, 0] != abi.DIAG_UNRESOLVED],
                                         ordered=True)
    return b


def build_graph(attached):
    """depgraph.build_graph (depgraph.py:507-528) on the GPU."""
    ns = _ns(attached)
    k = _kern(attached)
    b = _build(k)
    edges = _edges(ns, k.ks, b["bprod"], b["bcons"], b["bmeta"])
    diags = tuple(attached.diagnostics) + tuple(attached.cfg.diagnostics) + tuple(b["unresolved"]) \
        + tuple(b["sync_diags"])
    g = ns.DependencyGraph(attached, edges, diags)
    _graphs.put(g, b["edges"])
    return g


_reach_of: dict = {}      # id(result) -> result, the last few reaching_definitions results


def _remember_reach(res):
    _reach_of[id(res)] = res
    while len(_reach_of) > 16:
        _reach_of.pop(next(iter(_reach_of)))
    return res


def _unit_keys(ns, ks):
    """dense unit id -> (RegClass, index) (depgraph.py:41)"""
    rcs = [ns.RegClass(v) for v in E.REG_CLASSES]
    base = [int(x) for x in ks.unit_base] + [ks.n_units]
    keys = [None] * ks.n_units
    for c in range(7):
        for u in range(base[c], min(base[c + 1], ks.n_units)):
            keys[u] = (rcs[c], u - base[c])
    return keys


def reaching_definitions(cfg):
    """depgraph.reaching_definitions (depgraph.py:135-177): block-entry reach-in
    sets {(RegClass, index): frozenset(def indices)} for every block, computed by
    the device's reaching-definition search on every (block, unit) pair."""
    ns = _ns(cfg)
    k = _kern(cfg)
    B, U = k.ks.n_blocks, k.ks.n_units
    off, defs = ops.reach_in(k.dk)
    keys = _unit_keys(ns, k.ks)
    res = []
    for b in range(B):
        d = {}
        row = off[b * U:(b + 1) * U + 1]
        for u in np.flatnonzero(np.diff(row)).tolist():
            d[keys[u]] = frozenset(defs[row[u]:row[u + 1]].tolist())
        res.append(d)
    return _remember_reach(res)


def per_use_link(cfg, reach_in):
    """depgraph.per_use_link (depgraph.py:188-223): (links, unresolved-use
    diagnostics).  The device derives the reach-in sets itself (the same search
    reaching_definitions runs); `reach_in` must be reaching_definitions(cfg).
    Links are returned in build_graph's (consumer, producer, kind, register)
    order."""
    if _reach_of.get(id(reach_in)) is not reach_in and reach_in != reaching_definitions(cfg):
        raise ValueError("per_use_link: reach_in is not reaching_definitions(cfg) (the device "
                         "derives the reaching definitions itself)")
    ns = _ns(cfg)
    k = _kern(cfg)
    b = _build(k)
    r = b["n_regular"]
    edges = _edges(ns, k.ks, b["bprod"][:r], b["bcons"][:r], b["bmeta"][:r])
    return [ns.UseLink(e.producer, e.consumer, e.register, e.kind) for e in edges], list(b["unresolved"])


def liveness_filter(cfg, links):
    """depgraph.liveness_filter (depgraph.py:274-293) on the GPU: backward
    liveness fixed point, then the per-link live-out test."""
    links = list(links)
    if not links:
        return []
    k = _kern(cfg)
    prod = np.fromiter((l.producer for l in links), np.int32, len(links))
    cons = np.fromiter((l.consumer for l in links), np.int32, len(links))
    meta = np.fromiter((_ref27(l.register) | (E.EK_IDX[l.kind.value] << 27) for l in links), np.uint32,
                       len(links))
    keep = ops.liveness_filter(k.dk, prod, cons, meta)
    return [l for l, x in zip(links, keep.tolist()) if x]


def _sync_part(cfg, dialect):
    ns = _ns(cfg)
    if cfg.dialect.value != dialect:
        return [], []
    k = _kern(cfg)
    b = _build(k)
    r = b["n_regular"]
    return list(_edges(ns, k.ks, b["bprod"][r:], b["bcons"][r:], b["bmeta"][r:])), list(b["sync_diags"])


def trace_waitcnt(cfg):
    """depgraph.trace_waitcnt (depgraph.py:402-416): amd s_waitcnt edges."""
    return _sync_part(cfg, "amd")


def trace_barriers(cfg):
    """depgraph.trace_barriers (depgraph.py:446-463): nvidia barrier edges."""
    return _sync_part(cfg, "nvidia")


def trace_swsb(cfg):
    """depgraph.trace_swsb (depgraph.py:466-482): intel SBID edges."""
    return _sync_part(cfg, "intel")


def dump_graph(graph):
    """depgraph.dump_graph (depgraph.py:531-544): golden text, one edge per
    line sorted by (consumer, producer, kind) (host formatting)."""
    cfg = graph.cfg
    d = cfg.dialect.value
    lines = []
    for e in sorted(graph.edges, key=lambda e: (e.consumer, e.producer, e.kind.value)):
        reg = ""
        if e.register is not None:
            reg = " reg=" + diagnostics.format_register(d, E.RC_IDX[e.register.reg_class.value],
                                                        e.register.index, e.register.span)
        lines.append(f"0x{cfg.instructions[e.producer].offset:04x} -> "
                     f"0x{cfg.instructions[e.consumer].offset:04x} "
                     f"kind={e.kind.value}{reg} class={e.dep_class.value}")
    return "\n".join(lines) + ("\n" if lines else "")


# --------------------------------------------------------------------------
# pruning (analysis.py:143-314)

def _prune(graph, cfg: abi.LeoConfig):
    """One leo_prune call over the graph's device edges: the stages in
    cfg.stage_mask applied to every edge (each stage is a per-edge predicate,
    so one pass equals the reference's sequence of passes)."""
    ns = _ns(graph.attached)
    k = _kern(graph.attached)
    r, d = ops.prune(k.dk, k.dp, cfg, _dev_edges(graph))
    edges = _edges(ns, k.ks, r["pprod"], r["pcons"], r["pmeta"], r["npaths"], r["first"], r["plen"], r["pacc"])
    diags = diagnostics.render(k.ks.dialect, k.ks.offset, r["diag_records"], ordered=True)
    g = graph.with_edges(edges, tuple(diags))
    _graphs.put(g, d)
    return g


def run_pruning(graph, config):
    """analysis.run_pruning (analysis.py:302-314): stages 1 -> 2 -> 3 -> 4 per
    config.stage_mask (stage 4 only with prune_exec), one device pass."""
    return _prune(graph, _config_of(config, graph.cfg.dialect.value))


def prune_opcode(graph):
    """analysis.prune_opcode (analysis.py:143-162)."""
    return _prune(graph, abi.make_config(stage_mask=(1,), dialect=graph.cfg.dialect.value))


def prune_barrier(graph):
    """analysis.prune_barrier (analysis.py:165-185): nvidia only (identity otherwise)."""
    if graph.cfg.dialect.value != "nvidia":
        return graph
    return _prune(graph, abi.make_config(stage_mask=(2,), dialect="nvidia"))


def prune_latency(graph, table, max_paths=64, max_depth=512):
    """analysis.prune_latency (analysis.py:256-286)."""
    th = E.dense_thresholds((c.value, v) for c, v in table.thresholds)
    return _prune(graph, abi.make_config(stage_mask=(3,), thresholds=th, max_paths=max_paths,
                                         max_depth=max_depth, dialect=graph.cfg.dialect.value))


def prune_execution(graph, enabled):
    """analysis.prune_execution (analysis.py:289-299): identity when disabled."""
    if not enabled:
        return graph
    return _prune(graph, abi.make_config(stage_mask=(4,), prune_exec=True,
                                         dialect=graph.cfg.dialect.value))


# --------------------------------------------------------------------------
# blame (analysis.py:320-484), chains and coverage (:491-561)

def attribute_blame(graph, base_graph=None):
    """analysis.attribute_blame (analysis.py:431-484) on the GPU, for any
    graph; base_graph (the unpruned graph) feeds the indirect-addressing test."""
    ns = _ns(graph.attached)
    k = _kern(graph.attached)
    r = ops.blame(k.dk, k.dp, _dev_edges(graph), _dev_edges(base_graph) if base_graph is not None else None)
    return _entries(ns, k.ks, r, graph.edges)


def _entries(ns, ks, r, edges):
    subs = [ns.SelfBlame(v) for v in E.SELF_BLAMES]
    out = []
    regs = {}
    for s, e, sub, bl, f in zip(r["e_stalled"].tolist(), r["e_edge"].tolist(),
                                r["e_sub"].tolist(), r["e_blame"].tolist(),
                                r["e_factors"].tolist()):
        if e < 0:
            out.append(ns.BlameEntry(stalled=s, cause=None, kind=None, subcategory=subs[sub],
                                     blame_cycles=bl, factors=None))
        else:
            ed = edges[e]
            reg = None
            if ed.register is not None:
                rr = ed.register
                reg = regs.get(rr)
                if reg is None:
                    reg = regs[rr] = diagnostics.format_register(
                        ks.dialect, E.RC_IDX[rr.reg_class.value], rr.index, rr.span)
            out.append(ns.BlameEntry(stalled=s, cause=ed.producer, kind=ed.kind, subcategory=None,
                                     blame_cycles=bl, factors=ns.Factors(*f), register=reg))
    return out


def self_blame(index, attached, base_graph=None):
    """analysis.self_blame (analysis.py:414-428): the SELF entry of any
    instruction (S_j may be 0), classified on the device."""
    ns = _ns(attached)
    k = _kern(attached)
    if not 0 <= int(index) < k.ks.n_instr:
        raise IndexError(index)
    sub, cyc = ops.self_blame(k.dk, k.dp, _dev_edges(base_graph) if base_graph is not None else None,
                              [int(index)])
    return ns.BlameEntry(stalled=int(index), cause=None, kind=None,
                         subcategory=ns.SelfBlame(E.SELF_BLAMES[int(sub[0])]), blame_cycles=float(cyc[0]),
                         factors=None)


def _entry_arrays(blame):
    n = len(blame)
    st_ = np.fromiter((b.stalled for b in blame), np.int32, n)
    ca = np.fromiter((-1 if b.cause is None else b.cause for b in blame), np.int32, n)
    bl = np.fromiter((b.blame_cycles for b in blame), np.float64, n)
    return st_, ca, bl


def trace_chain(graph, blame, start, max_depth=32):
    """analysis.trace_chain (analysis.py:499-538): greedy backward walk along
    the highest-blame entry, on the device."""
    ns = _ns(graph.attached)
    if start >= len(graph.cfg.instructions) or start < 0:
        raise ValueError(f"chain start index {start} is not in the graph")
    blame = list(blame)
    chain = [ns.ChainHop(index=start, kind=None, blame_cycles=None, share=None, self_blame=None)]
    if max_depth <= 1:
        return chain
    k = _kern(graph.attached)
    _, ent, self_e = ops.trace_chain(k.dk, *_entry_arrays(blame), start, max_depth)
    attached = graph.attached
    for t in range(1, len(ent)):
        b = blame[ent[t]]
        s_node = attached.stall_cycles_at(chain[-1].index)
        chain.append(ns.ChainHop(index=b.cause, kind=b.kind, blame_cycles=b.blame_cycles,
                                 share=(b.blame_cycles / s_node) if s_node else None, self_blame=None))
    if self_e >= 0:
        chain[-1] = dataclasses.replace(chain[-1], self_blame=blame[self_e].subcategory)
    return chain


def single_dep_coverage(graph):
    """analysis.single_dep_coverage (analysis.py:547-561) on the device."""
    ns = _ns(graph.attached)
    if not graph.edges:
        return ns.Coverage(value=1.0, vacuous=True)
    nodes, qual = ops.coverage(_kern(graph.attached).dk, _dev_edges(graph))
    return ns.Coverage(value=qual / nodes, vacuous=False)


def rank_hotspots(attached, top_n, include_unsampled=False):
    """report.rank_hotspots (report.py:96-109) on the device (top_n <= 4096)."""
    top_n = max(0, int(top_n))
    if top_n == 0:
        return []
    k = _kern(attached)
    return ops.rank_hotspots(k.dk, k.dp, top_n, include_unsampled)


# --------------------------------------------------------------------------
# the slice and the per-line rollup (the two products the reference lacks)

def backward_slice(graph):
    """Multi-source backward slice from every instruction with S_j > 0 over
    graph.incoming: (members, {index: hop level})."""
    k = _kern(graph.attached)
    lv = ops.slice_levels(k.dk, k.dp, _dev_edges(graph))
    idx = np.flatnonzero(lv >= 0)
    return frozenset(idx.tolist()), {int(i): int(lv[i]) for i in idx}


def line_blame(graph, blame=None):
    """Per-source-line rollup: blame cycles by the cause's line
    (self entries: the stalled instruction's line) and stall cycles by the
    stalled instruction's line, keyed `file:line` / `<unknown>`.  `blame`:
    the entries to roll up (default: attribute_blame(graph) on the device)."""
    k = _kern(graph.attached)
    keys = k.ks.lines
    if blame is None:
        r = ops.blame(k.dk, k.dp, _dev_edges(graph), None, lines=True)
        lb, ls = r["line_blame"], r["line_stall"]
    else:
        lb, ls = ops.line_rollup(k.dk, k.dp, *_entry_arrays(list(blame)))
    return ({keys[i]: float(lb[i]) for i in np.flatnonzero(lb)},
            {keys[i]: float(ls[i]) for i in np.flatnonzero(ls)})


# --------------------------------------------------------------------------
# fused pass

def analyze(attached, config=None):
    """Fused build -> prune -> blame -> slice -> lines in one device pass
    (leo_analyze): (base graph, pruned graph, blame entries, slice,
    (line blame, line stall))."""
    ns = _ns(attached)
    ks, prof = soa.encode_attached(attached)
    r = device.analyze_soa(ks, prof, _config_of(config, ks.dialect), device=_dev())
    bdiag, pdiag = _split_diags(ks, r)
    prefix = tuple(attached.diagnostics) + tuple(attached.cfg.diagnostics)
    base = ns.DependencyGraph(attached, _edges(ns, ks, r["bprod"], r["bcons"], r["bmeta"]),
                              prefix + tuple(bdiag))
    pruned = ns.DependencyGraph(attached, _edges(ns, ks, r["pprod"], r["pcons"], r["pmeta"], r["npaths"],
                                                 r["first"], r["plen"], r["pacc"]),
                                prefix + tuple(bdiag) + tuple(pdiag))
    entries = _entries(ns, ks, r, pruned.edges)
    lv = r["level"]
    idx = np.flatnonzero(lv >= 0)
    keys = ks.lines
    lb, ls = r["line_blame"], r["line_stall"]
    lines = ({keys[i]: float(lb[i]) for i in np.flatnonzero(lb)},
             {keys[i]: float(ls[i]) for i in np.flatnonzero(ls)})
    return base, pruned, entries, (frozenset(idx.tolist()), {int(i): int(lv[i]) for i in idx}), lines


# --------------------------------------------------------------------------
# SoA session: host buffers in, host results out (the bench's e2e path)

class Session:
    """Analyse raw PC-sample streams for one kernel shape.  Each `analyze`
    call copies the kernel SoA, profile metadata and raw samples from (pinned)
    host memory, runs the fused device pipeline and reads back the blame
    entries and per-line totals."""

    H2D_FIELDS = device.K_ARRAYS

    def __init__(self, ks: soa.KernelSoA, prof_meta: soa.ProfileSoA, n_samples: int,
                 config: abi.LeoConfig | None = None, dev=None, pin: bool = True):
        self.dev = torch.device(dev) if dev is not None else _dev()
        self.ks = ks
        self.n_samples = int(n_samples)
        self.cfg = config or abi.make_config(dialect=ks.dialect)
        self.dk = device.DeviceKernel(ks, self.dev)
        self.dp = device.DeviceProfile(prof_meta, ks.n_instr, self.dev)
        # raw samples travel packed (one u32 word per sample, pc << 8 | category:
        # 4 bytes instead of 5) when every pc fits 24 bits and the stream is
        # long enough for the one-pass hashed binning
        self.packed = ks.n_instr < (1 << 24) and n_samples >= device.PACK_MIN_SAMPLES
        # 3 bytes per sample (pc << cat_bits | category) when the pcs and the
        # dialect's category ids fit 24 bits together (4 category bits for
        # NVIDIA / AMD, 5 for Intel): a quarter less over PCIe
        self.pack_width = 4
        self.cat_bits = device.cat_bits_for(len(E.vendor_categories(ks.dialect)))
        if (self.packed and self.cat_bits and ks.n_instr <= (1 << (24 - self.cat_bits))
                and not os.environ.get("LEO_PACK4")):
            self.pack_width = 3
        if self.packed and self.pack_width == 3:
            self.words = torch.empty((3 * n_samples + 3) & ~3, dtype=torch.uint8, device=self.dev)
        elif self.packed:
            self.words = torch.empty(max(n_samples, 1), dtype=torch.int32, device=self.dev)
        else:
            self.pc = torch.empty(max(n_samples, 1), dtype=torch.int32, device=self.dev)
            self.cat = torch.empty(max(n_samples, 1), dtype=torch.uint8, device=self.dev)
        self.lut = torch.empty(256, dtype=torch.uint8, device=self.dev)
        self.pin = pin
        self._host = {}
        self.h_pack = None
        if pin:
            self._pack_inputs()
        if self.packed and self.pack_width == 3:
            self.ds = device.DeviceSamples.from_packed(self.words, self.lut, n=n_samples, width=3,
                                                       cat_bits=self.cat_bits)
        elif self.packed:
            self.ds = device.DeviceSamples.from_packed(self.words[:n_samples], self.lut)
        else:
            self.ds = device.DeviceSamples.from_tensors(self.pc[:n_samples], self.cat[:n_samples], self.lut)
        self.an = device.Analyzer(self.dk, self.dev)
        self.use_graph = True
        self.graph = None

    def _pack_inputs(self):
        """Re-home every per-call input (kernel SoA, line ids, profile
        metadata, category table) into one device buffer mirrored by one
        pinned host buffer, so a call's H2D is a single copy instead of one
        per array.  Raw samples stay separate (the library pulls them on the
        binning branch)."""
        dk, dp = self.dk, self.dp
        specs = [("k_" + n, dk.t[n]) for n in self.H2D_FIELDS]
        if "seg_block" in dk.t:
            specs.append(("k_seg_block", dk.t["seg_block"]))
        specs.append(("line_id", dk.line_id))
        specs += [("p_" + n, getattr(dp, n)) for n in ("exec_cnt", "total", "eff", "sampled")]
        specs.append(("lut", self.lut))
        layout, off = [], 0
        for name, t in specs:
            nb = t.numel() * t.element_size()
            layout.append((name, off, nb, t))
            off = (off + nb + 15) & ~15
        self.d_pack = torch.empty(max(off, 16), dtype=torch.uint8, device=self.dev)
        self.h_pack = torch.empty(max(off, 16), dtype=torch.uint8).pin_memory()
        for name, o, nb, t in layout:
            dv = self.d_pack[o:o + nb].view(t.dtype).view(t.shape)
            dv.copy_(t)
            self._host[name] = self.h_pack[o:o + nb].view(t.dtype).view(t.shape)
            if name.startswith("k_"):
                dk.t[name[2:]] = dv
            elif name == "line_id":
                dk.line_id = dv
            elif name.startswith("p_"):
                setattr(dp, name[2:], dv)
            else:
                self.lut = dv
        dk.struct = abi.kernel_struct(dk.ks, lambda n: dk.t[n].data_ptr())
        dp.struct = abi.LeoProfile(dp.period, device.ptr(dp.lat), device.ptr(dp.cls_cnt), device.ptr(dp.exec_cnt),
                                   device.ptr(dp.total), device.ptr(dp.eff), device.ptr(dp.sampled))

    def _h(self, name, arr):
        """pinned host staging copy of a numpy input"""
        a = np.ascontiguousarray(arr)
        if a.dtype == np.uint32:
            a = a.view(np.int32)
        t = self._host.get(name)
        if t is None or t.numel() != a.size:
            t = torch.from_numpy(a.copy()).reshape(-1)
            if self.pin:
                t = t.pin_memory()
            self._host[name] = t
        else:
            t.numpy().reshape(a.shape)[...] = a
        return t

    def _check_sizes(self, ks, prof_meta, pc, cat, lut):
        """The captured graph copies from buffers sized at construction: a step
        whose arrays have other sizes is refused, not silently mis-copied."""
        n = self.ks.n_instr
        want = {"k_" + f: np.asarray(getattr(self.ks, f)).size for f in self.H2D_FIELDS}
        got = {"k_" + f: np.asarray(getattr(ks, f)).size for f in self.H2D_FIELDS}
        if getattr(self.ks, "seg_block", None) is not None or getattr(ks, "seg_block", None) is not None:
            want["k_seg_block"] = np.asarray(getattr(self.ks, "seg_block", ())).size
            got["k_seg_block"] = np.asarray(getattr(ks, "seg_block", ())).size
        want["line_id"], got["line_id"] = n, np.asarray(ks.line_id).size
        for f in ("exec_cnt", "total", "eff", "sampled"):
            want["p_" + f], got["p_" + f] = n, np.asarray(getattr(prof_meta, f)).size
        want["pc"], got["pc"] = self.n_samples, np.asarray(pc).size
        want["cat"], got["cat"] = self.n_samples, np.asarray(cat).size
        want["lut"], got["lut"] = 256, np.asarray(lut).size
        bad = {k: (got[k], v) for k, v in want.items() if got[k] != v}
        if bad:
            raise ValueError(f"Session.stage: input sizes differ from the session's shape "
                             f"(got, expected): {bad}")

    def stage(self, ks, prof_meta, pc, cat, lut):
        """Put one step's inputs into pinned host buffers (outside timing)."""
        self._check_sizes(ks, prof_meta, pc, cat, lut)
        for n in self.H2D_FIELDS:
            self._h("k_" + n, getattr(ks, n))
        if getattr(ks, "seg_block", None) is not None:
            self._h("k_seg_block", ks.seg_block)
        self._h("line_id", ks.line_id)
        for n in ("exec_cnt", "total", "eff", "sampled"):
            self._h("p_" + n, getattr(prof_meta, n))
        self._h("lut", lut)
        # the library copies the sample stream itself, on the binning branch
        if self.packed and self.pack_width == 3:
            if not device.packable24(pc, cat, self.ks.n_instr, self.cat_bits):
                raise ValueError("Session.stage: sample pc out of range (negative or >= n_instr) "
                                 f"or category id >= {1 << self.cat_bits}")
            self._h("words", device.pack_samples24(pc, cat, self.cat_bits))
            self.ds.set_host_packed(self._host["words"])
        elif self.packed:
            if not device.packable(pc):
                raise ValueError("Session.stage: sample pc out of range (negative or >= 2^24)")
            self._h("words", device.pack_samples(pc, cat).view(np.int32))
            self.ds.set_host_packed(self._host["words"])
        else:
            self._h("pc", pc)
            self._h("cat", cat)
            self.ds.set_host_sources(self._host["pc"], self._host["cat"].view(torch.uint8))

    def h2d_bytes(self) -> int:
        if self.h_pack is not None:
            names = ("words",) if self.packed else ("pc", "cat")
            return self.h_pack.numel() + sum(self._host[n].numel() * self._host[n].element_size() for n in names)
        return sum(t.numel() * t.element_size() for t in self._host.values())

    def _h2d(self):
        if self.h_pack is not None:
            self.d_pack.copy_(self.h_pack, non_blocking=True)
            return
        for n in self.H2D_FIELDS:
            self.dk.t[n].view(-1).copy_(self._host["k_" + n], non_blocking=True)
        if "k_seg_block" in self._host:
            self.dk.t["seg_block"].view(-1).copy_(self._host["k_seg_block"], non_blocking=True)
        self.dk.line_id.copy_(self._host["line_id"], non_blocking=True)
        for n in ("exec_cnt", "total", "eff", "sampled"):
            getattr(self.dp, n).copy_(self._host["p_" + n], non_blocking=True)
        self.lut.copy_(self._host["lut"], non_blocking=True)

    def _pinned(self, like: torch.Tensor) -> torch.Tensor:
        return torch.empty(like.shape, dtype=like.dtype).pin_memory()

    def _capture(self):
        """Size the buffers with an eager run, then capture one CUDA graph:
        H2D of the kernel SoA and profile metadata, the fused pipeline (whose
        binning branch pulls the pinned sample stream while the graph is being
        built), the sparse per-line list (leo_line_compact), and D2H of the
        counters, the touched lines and the blame entries."""
        self._h2d()
        self.an.run(self.dp, self.cfg, self.ds)
        self.an.ensure_workspace()
        self.an.run(self.dp, self.cfg, self.ds)
        an = self.an
        L = int(an.line_blame.numel())
        self.n_lines = L
        self.d_lid = torch.empty(max(L, 1), dtype=torch.int32, device=self.dev)
        self.d_lb = torch.empty(max(L, 1), dtype=torch.float64, device=self.dev)
        self.d_ls = torch.empty(max(L, 1), dtype=torch.float64, device=self.dev)
        self.d_lcnt = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._compact_lines()
        torch.cuda.synchronize(self.dev)
        self.h_ctr = self._pinned(an.ctr)
        self.h_lcnt = self._pinned(self.d_lcnt)
        self.h_lid = self._pinned(self.d_lid)
        self.h_lb = self._pinned(self.d_lb)
        self.h_ls = self._pinned(self.d_ls)
        cap = an.caps.blame
        # blame entries and touched lines: the graph copies prefixes sized from
        # this sizing run (the counts are device values); a longer result
        # copies its tail after the replay
        nbl0 = int(an.counts()[device.C_BLAME])
        self.k_pre = min(cap, int(nbl0 * 1.1) + 256)
        nl0 = int(self.d_lcnt.item())
        self.l_pre = min(max(L, 1), int(nl0 * 1.1) + 256)
        self.h_ent = {name: torch.empty(cap * w, dtype=getattr(an, src).dtype).pin_memory()
                      for name, src, w in self.ENTRY_FIELDS}
        # numpy views of the pinned read-back buffers (no per-call tensor ops)
        self.n_ctr, self.n_lcnt = self.h_ctr.numpy(), self.h_lcnt.numpy()
        self.n_lid, self.n_lb, self.n_ls = self.h_lid.numpy(), self.h_lb.numpy(), self.h_ls.numpy()
        self.n_ent = {name: t.numpy() for name, t in self.h_ent.items()}
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        torch.cuda.synchronize(self.dev)
        with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
            self._h2d()
            an.launch(self.dp, self.cfg, self.ds)
            self._compact_lines()
            self.h_ctr.copy_(an.ctr, non_blocking=True)
            self.h_lcnt.copy_(self.d_lcnt, non_blocking=True)
            self._copy_lines(0, self.l_pre)
            self._copy_entries(0, self.k_pre)
        torch.cuda.synchronize(self.dev)
        self.graph = g

    def _compact_lines(self):
        L = self.n_lines
        rc = _lib.lib().leo_line_compact(device.ptr(self.an.line_blame), device.ptr(self.an.line_stall), L, L,
                                         device.ptr(self.d_lid), device.ptr(self.d_lb), device.ptr(self.d_ls),
                                         device.ptr(self.d_lcnt),
                                         torch.cuda.current_stream(self.dev).cuda_stream)
        _lib.check(rc, "leo_line_compact")

    def _copy_lines(self, lo, hi):
        for h, d in ((self.h_lid, self.d_lid), (self.h_lb, self.d_lb), (self.h_ls, self.d_ls)):
            h[lo:hi].copy_(d[lo:hi], non_blocking=True)

    # self-contained blame entries read back per call: stalled, cause (-1 =
    # self), the cause edge's meta word (kind, dep class, register), SelfBlame
    # subcategory, blame cycles and the four Eq. 1 factors (53 bytes each)
    ENTRY_FIELDS = (("e_stalled", "bl_stalled", 1), ("e_cause", "bl_cause", 1), ("e_meta", "bl_meta", 1),
                    ("e_sub", "bl_sub", 1), ("e_blame", "bl_blame", 1), ("e_factors", "bl_factors", 4))

    def _copy_entries(self, lo, hi):
        for name, src, w in self.ENTRY_FIELDS:
            self.h_ent[name][lo * w:hi * w].copy_(getattr(self.an, src)[lo * w:hi * w], non_blocking=True)

    def _entry_bytes(self, n):
        return sum(n * w * self.h_ent[name].element_size() for name, _, w in self.ENTRY_FIELDS)

    @staticmethod
    def dense_lines(r: dict, n_lines: int):
        """(line_blame, line_stall) as dense f64[n_lines] vectors from a result."""
        lb = np.zeros(n_lines)
        ls = np.zeros(n_lines)
        lb[r["line_ids"]] = r["line_blame"]
        ls[r["line_ids"]] = r["line_stall"]
        return lb, ls

    def _result(self, ent, nbl, lid, lb, ls, copy):
        cp = (lambda a: a.copy()) if copy else (lambda a: a)
        out = {name: cp(ent[name][:nbl * w]) for name, _, w in self.ENTRY_FIELDS}
        out["e_meta"] = out["e_meta"].view(np.uint32)
        out["e_factors"] = out["e_factors"].reshape(-1, 4)
        out["line_ids"], out["line_blame"], out["line_stall"] = cp(lid), cp(lb), cp(ls)
        return out

    def analyze(self, allreduce=None, copy: bool = False):
        """Copy staged inputs in, run, copy results out.  Returns a host dict
        of self-contained blame entries (e_stalled, e_cause, e_meta, e_sub,
        e_blame, e_factors) and the touched source lines (line_ids ascending,
        with their line_blame / line_stall totals; `dense_lines` expands them).
        The arrays are views of the session's pinned read-back buffers, valid
        until the next call (`copy=True` returns owned copies).
        `allreduce(line_blame, line_stall)` (multi-GPU) runs on the device
        line vectors before they are read back.  Single-GPU calls replay one
        CUDA graph (H2D + pipeline + D2H of counters, touched lines and the
        entries' expected prefix); longer results read back their tail."""
        if allreduce is None and self.use_graph:
            self.submit()
            r = self._collect_graph(copy)
            if r is not None:
                return r
        return self._analyze_eager(allreduce, copy)

    def submit(self, stream: torch.cuda.Stream | None = None):
        """Start one call without waiting for it: replay the session's CUDA
        graph (H2D, pipeline, D2H prefixes) on `stream` (default: the current
        stream).  `collect()` waits and returns the result.  Sessions submitted
        on different streams overlap each other's transfers and compute (a
        batch of kernels: one call's read-back beside the next one's upload)."""
        if getattr(self, "graph", None) is None:
            self._capture()
        self._stream = stream if stream is not None else torch.cuda.current_stream(self.dev)
        with torch.cuda.stream(self._stream):
            self.graph.replay()

    def collect(self, copy: bool = False):
        """The result of the last `submit()` (as `analyze()` returns it)."""
        r = self._collect_graph(copy)
        return r if r is not None else self._analyze_eager(None, copy)

    def _collect_graph(self, copy):
        st = self._stream
        st.synchronize()
        c = self.n_ctr
        nbl = int(c[device.C_BLAME])
        nl = int(self.n_lcnt[0])
        if c[device.C_STATUS] == 0 and nbl <= self.an.caps.blame and nl <= self.n_lines:
            if nbl > self.k_pre or nl > self.l_pre:   # tails beyond the in-graph prefixes
                with torch.cuda.stream(st):
                    if nbl > self.k_pre:
                        self._copy_entries(self.k_pre, nbl)
                    if nl > self.l_pre:
                        self._copy_lines(self.l_pre, nl)
                st.synchronize()
            self.last_d2h = (c.nbytes + 4 + 20 * max(nl, self.l_pre)
                             + self._entry_bytes(max(nbl, self.k_pre)))
            return self._result(self.n_ent, nbl, self.n_lid[:nl], self.n_lb[:nl], self.n_ls[:nl], copy)
        self.graph = None                  # overflow: grow eagerly, recapture next call
        return None

    def _analyze_eager(self, allreduce, copy):
        self._h2d()
        self.an.launch(self.dp, self.cfg, self.ds)
        c = self.an.ctr.cpu().numpy()          # sync: how much to read back
        self.an.ensure_workspace()             # persistent scratch for the next call
        nbl = min(int(c[device.C_BLAME]), self.an.caps.blame)
        if int(c[device.C_BLAME]) > self.an.caps.blame or c[device.C_STATUS] != 0:
            self.an.run(self.dp, self.cfg, self.ds)
            c = self.an.ctr.cpu().numpy()
            nbl = int(c[device.C_BLAME])
        if allreduce is not None:
            allreduce(self.an.line_blame, self.an.line_stall)
        ent = {name: getattr(self.an, src)[:nbl * w].to("cpu", non_blocking=True)
               for name, src, w in self.ENTRY_FIELDS}
        lb = self.an.line_blame.to("cpu", non_blocking=True)
        ls = self.an.line_stall.to("cpu", non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        self.last_d2h = (sum(t.numel() * t.element_size() for t in ent.values()) + c.nbytes
                         + lb.numel() * 8 + ls.numel() * 8)
        lbn, lsn = lb.numpy(), ls.numpy()
        lid = np.flatnonzero((lbn != 0) | (lsn != 0)).astype(np.int32)
        return self._result({k: v.numpy() for k, v in ent.items()}, nbl, lid, lbn[lid], lsn[lid], True)


# --------------------------------------------------------------------------
# report assembly on device outputs (report.py:128-213)

def build_report_soa(ks, prof, config, meta, top_n: int = 10, include_unsampled: bool = False,
                     chain_depth: int = 32, samples=None, dev=None, R=None):
    """StallReport of one kernel given as SoA + ReportMeta (the analysis, the
    coverage, the ranking, the cause order and the chains run on the device;
    the host formats)."""
    dev = torch.device(dev) if dev is not None else _dev()
    dk = device.DeviceKernel(ks, dev)
    dp = device.DeviceProfile(prof, ks.n_instr, dev)
    ds = device.DeviceSamples(*samples, dev) if samples is not None else None
    an = device.Analyzer(dk, dev)
    an.run(dp, _config_of(config, ks.dialect), ds)
    r = an.result()
    r["lat"] = dp.lat.cpu().numpy()
    r["cls_cnt"] = dp.cls_cnt.cpu().numpy().reshape(-1, 8)
    rep = an.report(dp, top_n, include_unsampled, chain_depth)
    bdiag, pdiag = _split_diags(ks, r)
    diags = tuple(ks.prefix_diagnostics) + tuple(bdiag) + tuple(pdiag)
    return report.assemble(ks, meta, r, rep, diags, R)


def build_report(cfg, profile, config, top_n: int = 10, include_unsampled: bool = False,
                 chain_depth: int = 32):
    """report.build_report (report.py:128-213) with the analysis and the report
    assembly on the GPU; takes and returns the reference's objects."""
    import sys
    attach = sys.modules[type(profile).__module__].attach      # profile.attach (profile.py)
    attached = attach(cfg, profile)
    ks, prof = soa.encode_attached(attached)
    meta = report.meta_from_reference(cfg, profile, config)
    return build_report_soa(ks, prof, config, meta, top_n, include_unsampled, chain_depth)
