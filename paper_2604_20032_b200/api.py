"""Public API: the reference analyzer's names and types, backed by the CUDA path.

Drop-in for the stalltrace hot path (`stalltrace/__init__.py:9-37`):

    build_graph(attached) -> DependencyGraph                 depgraph.py:507
    run_pruning(graph, config) -> DependencyGraph            analysis.py:302
    prune_opcode / prune_barrier / prune_latency / prune_execution   analysis.py:143-299
    attribute_blame(graph, base_graph=None) -> list[BlameEntry]      analysis.py:431
    self_blame(index, attached, base_graph=None) -> BlameEntry       analysis.py:414

plus the two hot-path products the reference does not have:

    backward_slice(graph) -> (frozenset[int], dict[int, int])
    line_blame(graph, blame) -> (dict[str, float], dict[str, float])

and `Session`, the SoA-level entry a profiling service uses (raw PC-sample
stream in, per-instruction blame entries + per-line totals out).

Inputs are the reference's own objects (duck-typed: any object with the
reference attribute names works); outputs are built from `stalltrace` classes
when that package is importable, else from the mirror classes in
`paper_2604_20032_b200.types` (same names, fields and enum values).  Every
computation runs on the GPU through libleo_b200.so; there is no CPU fallback.
"""

from __future__ import annotations

import dataclasses
import weakref

import numpy as np
import torch

from . import abi, device, diagnostics, report, soa, types
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
# one cached device analysis per (graph, config)

@dataclasses.dataclass
class _Analysis:
    ks: soa.KernelSoA
    prof: soa.ProfileSoA
    raw: dict


_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _config_of(config, dialect):
    if config is None:
        return abi.make_config(dialect=dialect)
    if isinstance(config, abi.LeoConfig):
        return config
    return abi.config_from_reference(config, dialect)


def _run(attached, config=None) -> _Analysis:
    ks, prof = soa.encode_attached(attached)
    r = device.analyze_soa(ks, prof, _config_of(config, ks.dialect), device=_dev())
    return _Analysis(ks, prof, r)


def _edges(ns, ks, prod, cons, meta, npaths=None, first=None, plen=None, pacc=None):
    out = []
    cls = ns.RegClass
    rcs = [cls(v) for v in E.REG_CLASSES]
    kinds = [ns.EdgeKind(v) for v in E.EDGE_KINDS]
    dcs = [ns.DepClass(v) for v in E.DEP_CLASSES]
    prod, cons, meta = prod.tolist(), cons.tolist(), meta.astype(np.uint32).tolist()
    if npaths is not None:
        npaths, first, plen, pacc = npaths.tolist(), first.tolist(), plen.tolist(), pacc.tolist()
    for x in range(len(prod)):
        m = meta[x]
        kind = (m >> 27) & 7
        reg = None
        if kind < 2:
            reg = ns.RegisterRef(rcs[(m >> 24) & 7], m & 0xFFFF, (m >> 16) & 0xFF)
        paths = ()
        if npaths is not None and npaths[x] > 0:
            f = first[x]
            paths = tuple(ns.PathRecord(plen[f + q], pacc[f + q]) for q in range(npaths[x]))
        out.append(ns.DepEdge(producer=prod[x], consumer=cons[x], kind=kinds[kind], register=reg,
                              dep_class=dcs[(m >> 30) & 3], valid_paths=paths))
    return tuple(out)


def _graph(ns, attached, edges, diags, analysis, pruned):
    g = ns.DependencyGraph(attached, edges, tuple(diags))
    _cache[g] = (analysis, pruned)
    return g


def _split_diags(ks, r):
    recs = diagnostics.order(r["diag_records"])
    build = recs[recs[:, 0] != abi.DIAG_PATH_CAPPED] if recs.size else recs
    prune = recs[recs[:, 0] == abi.DIAG_PATH_CAPPED] if recs.size else recs
    return (diagnostics.render(ks.dialect, ks.offset, build, ordered=True),
            diagnostics.render(ks.dialect, ks.offset, prune, ordered=True))


# --------------------------------------------------------------------------
# reference-compatible functions

def build_graph(attached):
    """depgraph.build_graph (depgraph.py:507-528) on the GPU."""
    ns = _ns(attached)
    a = _run(attached, abi.make_config(stage_mask=(), dialect=attached.cfg.dialect.value))
    r = a.raw
    edges = _edges(ns, a.ks, r["bprod"], r["bcons"], r["bmeta"])
    bdiag, _ = _split_diags(a.ks, r)
    return _graph(ns, attached, edges, tuple(attached.diagnostics) + tuple(attached.cfg.diagnostics)
                  + tuple(bdiag), a, False)


def _prune_with(graph, config):
    attached = graph.attached
    ns = _ns(attached)
    a = _run(attached, config)
    r = a.raw
    base = _edges(ns, a.ks, r["bprod"], r["bcons"], r["bmeta"])
    if tuple((e.producer, e.consumer, e.kind, e.register) for e in base) != \
            tuple((e.producer, e.consumer, e.kind, e.register) for e in graph.edges):
        raise ValueError("graph was not produced by build_graph on this kernel; the device "
                         "pipeline prunes the build_graph edge list")
    edges = _edges(ns, a.ks, r["pprod"], r["pcons"], r["pmeta"], r["npaths"], r["first"],
                   r["plen"], r["pacc"])
    _, pdiag = _split_diags(a.ks, r)
    return _graph(ns, attached, edges, tuple(graph.diagnostics) + tuple(pdiag), a, True)


def run_pruning(graph, config):
    """analysis.run_pruning (analysis.py:302-314) on the GPU."""
    return _prune_with(graph, config)


def _stage(graph, mask, **kw):
    d = graph.cfg.dialect.value
    th = kw.pop("thresholds", None)
    return _prune_with(graph, abi.make_config(stage_mask=mask, thresholds=th, dialect=d, **kw))


def prune_opcode(graph):
    """analysis.prune_opcode (analysis.py:143-162)."""
    return _stage(graph, (1,))


def prune_barrier(graph):
    """analysis.prune_barrier (analysis.py:165-185)."""
    if graph.cfg.dialect.value != "nvidia":
        return graph
    return _stage(graph, (2,))


def prune_latency(graph, table, max_paths=64, max_depth=512):
    """analysis.prune_latency (analysis.py:256-286)."""
    th = E.dense_thresholds((c.value, v) for c, v in table.thresholds)
    return _stage(graph, (3,), thresholds=th, max_paths=max_paths, max_depth=max_depth)


def prune_execution(graph, enabled):
    """analysis.prune_execution (analysis.py:289-299)."""
    if not enabled:
        return graph
    return _stage(graph, (4,), prune_exec=True)


def attribute_blame(graph, base_graph=None):
    """analysis.attribute_blame (analysis.py:431-484) on the GPU.  When
    `graph` came from run_pruning the device result of that run is reused;
    base_graph (the unpruned graph) feeds the indirect-addressing test."""
    ns = _ns(graph.attached)
    hit = _cache.get(graph)
    if hit is None:
        raise ValueError("attribute_blame needs a graph produced by this package's "
                         "build_graph / run_pruning")
    a, pruned = hit
    r = a.raw
    ks = a.ks
    if not pruned:
        # blame directly on the base graph: prune with no stages (identity map)
        a = _run(graph.attached, abi.make_config(stage_mask=(), dialect=ks.dialect))
        r = a.raw
    return _entries(ns, ks, r, base_graph is not None)


def _entries(ns, ks, r, with_base=True):
    kinds = [ns.EdgeKind(v) for v in E.EDGE_KINDS]
    subs = [ns.SelfBlame(v) for v in E.SELF_BLAMES]
    out = []
    pprod, pmeta = r["pprod"].tolist(), r["pmeta"].astype(np.uint32).tolist()
    for s, e, sub, bl, f in zip(r["e_stalled"].tolist(), r["e_edge"].tolist(),
                                r["e_sub"].tolist(), r["e_blame"].tolist(),
                                r["e_factors"].tolist()):
        if e < 0:
            if not with_base and sub == E.SB_IDX["indirect_addressing"]:
                sub = E.SB_IDX["memory_latency"]
            out.append(ns.BlameEntry(stalled=s, cause=None, kind=None, subcategory=subs[sub],
                                     blame_cycles=bl, factors=None))
        else:
            m = pmeta[e]
            kind = (m >> 27) & 7
            reg = diagnostics.format_ref27(ks.dialect, m & 0x07FFFFFF) if kind < 2 else None
            out.append(ns.BlameEntry(stalled=s, cause=pprod[e], kind=kinds[kind], subcategory=None,
                                     blame_cycles=bl, factors=ns.Factors(*f), register=reg))
    return out


def self_blame(index, attached, base_graph=None):
    """analysis.self_blame (analysis.py:414-428): the SELF entry of one
    instruction (computed by the device blame kernel with no incoming edges)."""
    ns = _ns(attached)
    a = _run(attached, abi.make_config(stage_mask=(1, 2, 3, 4), dialect=attached.cfg.dialect.value))
    r = a.raw
    sel = np.flatnonzero((r["e_stalled"] == index) & (r["e_edge"] < 0))
    if sel.size:
        x = int(sel[0])
        sub = int(r["e_sub"][x])
    else:
        raise ValueError("self_blame: instruction has incoming edges or no stall cycles")
    if base_graph is None and sub == E.SB_IDX["indirect_addressing"]:
        sub = E.SB_IDX["memory_latency"]
    return ns.BlameEntry(stalled=index, cause=None, kind=None,
                         subcategory=ns.SelfBlame(E.SELF_BLAMES[sub]),
                         blame_cycles=float(r["e_blame"][x]), factors=None)


def backward_slice(graph):
    """Multi-source backward slice from every instruction with S_j > 0 over
    graph.incoming: (members, {index: hop level})."""
    hit = _cache.get(graph)
    if hit is None:
        raise ValueError("backward_slice needs a graph produced by this package")
    a, pruned = hit
    r = a.raw if pruned else _run(graph.attached, abi.make_config(stage_mask=(), dialect=a.ks.dialect)).raw
    lv = r["level"]
    idx = np.flatnonzero(lv >= 0)
    return frozenset(idx.tolist()), {int(i): int(lv[i]) for i in idx}


def line_blame(graph, blame=None):
    """Per-source-line rollup: blame cycles by the cause's
    line (self entries: the stalled instruction's line) and stall cycles by the
    stalled instruction's line, keyed `file:line` / `<unknown>`."""
    hit = _cache.get(graph)
    if hit is None:
        raise ValueError("line_blame needs a graph produced by this package")
    a, _ = hit
    keys = a.ks.lines
    lb, ls = a.raw["line_blame"], a.raw["line_stall"]
    return ({keys[i]: float(lb[i]) for i in np.flatnonzero(lb)},
            {keys[i]: float(ls[i]) for i in np.flatnonzero(ls)})


def analyze(attached, config=None):
    """Fused build -> prune -> blame -> slice -> lines in one device pass:
    (base graph, pruned graph, blame entries, slice, (line blame, line stall))."""
    ns = _ns(attached)
    a = _run(attached, config)
    r = a.raw
    bdiag, pdiag = _split_diags(a.ks, r)
    prefix = tuple(attached.diagnostics) + tuple(attached.cfg.diagnostics)
    base = _graph(ns, attached, _edges(ns, a.ks, r["bprod"], r["bcons"], r["bmeta"]),
                  prefix + tuple(bdiag), a, False)
    pruned = _graph(ns, attached, _edges(ns, a.ks, r["pprod"], r["pcons"], r["pmeta"], r["npaths"],
                                         r["first"], r["plen"], r["pacc"]),
                    prefix + tuple(bdiag) + tuple(pdiag), a, True)
    entries = _entries(ns, a.ks, r)
    return base, pruned, entries, backward_slice(pruned), line_blame(pruned)


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
        self.cfg = config or abi.make_config(dialect=ks.dialect)
        self.dk = device.DeviceKernel(ks, self.dev)
        self.dp = device.DeviceProfile(prof_meta, ks.n_instr, self.dev)
        self.pc = torch.empty(max(n_samples, 1), dtype=torch.int32, device=self.dev)
        self.cat = torch.empty(max(n_samples, 1), dtype=torch.uint8, device=self.dev)
        self.lut = torch.empty(256, dtype=torch.uint8, device=self.dev)
        self.pin = pin
        self._host = {}
        self.h_pack = None
        if pin:
            self._pack_inputs()
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

    def stage(self, ks, prof_meta, pc, cat, lut):
        """Put one step's inputs into pinned host buffers (outside timing)."""
        for n in self.H2D_FIELDS:
            self._h("k_" + n, getattr(ks, n))
        if getattr(ks, "seg_block", None) is not None:
            self._h("k_seg_block", ks.seg_block)
        self._h("line_id", ks.line_id)
        for n in ("exec_cnt", "total", "eff", "sampled"):
            self._h("p_" + n, getattr(prof_meta, n))
        self._h("pc", pc)
        self._h("cat", cat)
        self._h("lut", lut)
        # the library copies the sample stream itself, on the binning branch
        self.ds.set_host_sources(self._host["pc"], self._host["cat"].view(torch.uint8))

    def h2d_bytes(self) -> int:
        if self.h_pack is not None:
            return self.h_pack.numel() + sum(self._host[n].numel() * self._host[n].element_size() for n in ("pc", "cat"))
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
        built), and D2H of the counters and per-line vectors."""
        self._h2d()
        self.an.run(self.dp, self.cfg, self.ds)
        self.an.ensure_workspace()
        self.an.run(self.dp, self.cfg, self.ds)
        an = self.an
        self.h_ctr = self._pinned(an.ctr)
        self.h_lb = self._pinned(an.line_blame)
        self.h_ls = self._pinned(an.line_stall)
        cap = an.caps.blame
        # blame entries: the graph copies a prefix sized from this sizing run
        # (the count is a device value); a longer result copies its tail
        nbl0 = int(an.counts()[device.C_BLAME])
        self.k_pre = min(cap, int(nbl0 * 1.1) + 256)
        self.h_st = torch.empty(cap, dtype=torch.int32).pin_memory()
        self.h_ed = torch.empty(cap, dtype=torch.int32).pin_memory()
        self.h_bl = torch.empty(cap, dtype=torch.float64).pin_memory()
        # numpy views of the pinned read-back buffers (no per-call tensor ops)
        self.n_ctr, self.n_lb, self.n_ls = self.h_ctr.numpy(), self.h_lb.numpy(), self.h_ls.numpy()
        self.n_st, self.n_ed, self.n_bl = self.h_st.numpy(), self.h_ed.numpy(), self.h_bl.numpy()
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        torch.cuda.synchronize(self.dev)
        with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
            self._h2d()
            an.launch(self.dp, self.cfg, self.ds)
            self.h_ctr.copy_(an.ctr, non_blocking=True)
            self.h_lb.copy_(an.line_blame, non_blocking=True)
            self.h_ls.copy_(an.line_stall, non_blocking=True)
            k = self.k_pre
            self.h_st[:k].copy_(an.bl_stalled[:k], non_blocking=True)
            self.h_ed[:k].copy_(an.bl_edge[:k], non_blocking=True)
            self.h_bl[:k].copy_(an.bl_blame[:k], non_blocking=True)
        torch.cuda.synchronize(self.dev)
        self.graph = g

    def analyze(self, allreduce=None):
        """Copy staged inputs in, run, copy results out.  Returns host dict.
        `allreduce(line_blame, line_stall)` (multi-GPU) runs on the device line
        vectors before they are read back.  Single-GPU calls replay one CUDA
        graph (H2D + pipeline + D2H of counters and line vectors); the blame
        entries are then read back at their device-reported count."""
        if allreduce is None and self.use_graph:
            if getattr(self, "graph", None) is None:
                self._capture()
            self.graph.replay()
            torch.cuda.current_stream(self.dev).synchronize()
            c = self.n_ctr
            nbl = int(c[device.C_BLAME])
            if c[device.C_STATUS] == 0 and nbl <= self.an.caps.blame:
                an, k = self.an, self.k_pre
                if nbl > k:                       # tail beyond the in-graph prefix
                    self.h_st[k:nbl].copy_(an.bl_stalled[k:nbl], non_blocking=True)
                    self.h_ed[k:nbl].copy_(an.bl_edge[k:nbl], non_blocking=True)
                    self.h_bl[k:nbl].copy_(an.bl_blame[k:nbl], non_blocking=True)
                    torch.cuda.current_stream(self.dev).synchronize()
                self.last_d2h = (c.nbytes + self.h_lb.numel() * 8 + self.h_ls.numel() * 8
                                 + max(nbl, self.k_pre) * 16)
                return {"e_stalled": self.n_st[:nbl].copy(), "e_edge": self.n_ed[:nbl].copy(),
                        "e_blame": self.n_bl[:nbl].copy(), "line_blame": self.n_lb.copy(),
                        "line_stall": self.n_ls.copy()}
            self.graph = None                  # overflow: grow eagerly, recapture next call
        self._h2d()
        self.an.launch(self.dp, self.cfg, self.ds)
        c = self.an.ctr.cpu().numpy()          # sync: how much to read back
        self.an.ensure_workspace()             # persistent scratch for the next call
        nbl = min(int(c[device.C_BLAME]), self.an.caps.blame)
        if nbl > self.an.caps.blame or c[device.C_STATUS] != 0:
            self.an.run(self.dp, self.cfg, self.ds)
            c = self.an.ctr.cpu().numpy()
            nbl = int(c[device.C_BLAME])
        if allreduce is not None:
            allreduce(self.an.line_blame, self.an.line_stall)
        out = {
            "e_stalled": self.an.bl_stalled[:nbl].to("cpu", non_blocking=True),
            "e_edge": self.an.bl_edge[:nbl].to("cpu", non_blocking=True),
            "e_blame": self.an.bl_blame[:nbl].to("cpu", non_blocking=True),
            "line_blame": self.an.line_blame.to("cpu", non_blocking=True),
            "line_stall": self.an.line_stall.to("cpu", non_blocking=True),
        }
        torch.cuda.current_stream(self.dev).synchronize()
        self.last_d2h = sum(t.numel() * t.element_size() for t in out.values()) + c.nbytes
        return {k: v.numpy() for k, v in out.items()}


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
