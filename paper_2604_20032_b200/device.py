"""Device-resident SoA buffers and the stream-ordered pipeline driver.

PyTorch provides device memory and the stream; all compute is in
libleo_b200.so.  One `Analyzer` owns the output buffers (sized by capacity,
grown on overflow) so repeated runs reuse memory, as a serving process would.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import abi
from . import enums as E
from ._lib import check, lib

K_ARRAYS = ("opclass", "block_of", "opnd_ptr", "opnd", "sync_kind", "sync_a", "sync_b",
            "blk_first", "blk_last", "succ_ptr", "succ", "pred_ptr", "pred")
_TORCH_DT = {np.dtype(np.uint8): torch.uint8, np.dtype(np.int32): torch.int32,
             np.dtype(np.uint32): torch.int32, np.dtype(np.int64): torch.int64,
             np.dtype(np.float64): torch.float64}


def to_device(a: np.ndarray, device, pin: bool = False) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    if a.size == 0:
        return torch.zeros(1, dtype=_TORCH_DT[a.dtype], device=device)
    t = torch.from_numpy(a)
    return t.to(device, non_blocking=pin)


def ptr(t: torch.Tensor | None) -> int:
    return 0 if t is None else t.data_ptr()


class DeviceKernel:
    """KernelSoA uploaded to HBM."""

    def __init__(self, ks, device="cuda"):
        self.ks = ks
        self.device = torch.device(device)
        self.t = {n: to_device(getattr(ks, n), self.device) for n in K_ARRAYS}
        if getattr(ks, "seg_block", None) is not None:
            self.t["seg_block"] = to_device(np.asarray(ks.seg_block, dtype=np.int32), self.device)
        self.line_id = to_device(np.asarray(ks.line_id, dtype=np.int32), self.device)
        self.n_lines = int(len(ks.lines)) if ks.lines is not None else int(ks.line_id.max()) + 1
        self.struct = abi.kernel_struct(ks, lambda n: self.t[n].data_ptr())

    @property
    def n_instr(self):
        return self.ks.n_instr

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.t.values()) + self.line_id.numel() * 4


class DeviceProfile:
    """ProfileSoA in HBM.  lat / cls_cnt are writable (stage-0 binning output)."""

    def __init__(self, prof, n_instr: int, device="cuda"):
        dev = torch.device(device)
        self.period = int(prof.period)
        self.lat = to_device(np.asarray(prof.lat, dtype=np.int32), dev)
        self.cls_cnt = to_device(np.asarray(prof.cls_cnt, dtype=np.int32).reshape(-1), dev)
        self.exec_cnt = to_device(np.asarray(prof.exec_cnt, dtype=np.int64), dev)
        self.total = to_device(np.asarray(prof.total, dtype=np.int32), dev)
        self.eff = to_device(np.asarray(prof.eff, dtype=np.float64), dev)
        self.sampled = to_device(np.asarray(prof.sampled, dtype=np.uint8), dev)
        self.struct = abi.LeoProfile(self.period, ptr(self.lat), ptr(self.cls_cnt), ptr(self.exec_cnt),
                                     ptr(self.total), ptr(self.eff), ptr(self.sampled))


def pack_samples(pc, cat) -> np.ndarray:
    """The packed raw-sample stream (LeoSamples.packed, ABI v3): one u32 word
    per sample, pc << 8 | category."""
    return (np.asarray(pc).astype(np.uint32) << np.uint32(8)) | np.asarray(cat, dtype=np.uint8).astype(np.uint32)


def packable(pc) -> bool:
    pc = np.asarray(pc)
    return pc.size == 0 or (int(pc.min()) >= 0 and int(pc.max()) < (1 << 24))


def pack_samples24(pc, cat, cat_bits: int = 4) -> np.ndarray:
    """The 3-byte packed stream (LeoSamples.packed_bytes = 3, ABI v4): one
    little-endian 24-bit word per sample, pc << cat_bits | category, as 3 * S
    bytes (padded with zeros to a multiple of 4)."""
    w = ((np.asarray(pc).astype(np.uint32) << np.uint32(cat_bits))
         | np.asarray(cat, dtype=np.uint8).astype(np.uint32))
    n = w.shape[0]
    out = np.zeros((3 * n + 3) & ~3, dtype=np.uint8)
    out[:3 * n] = w.view(np.uint8).reshape(n, 4)[:, :3].reshape(-1)
    return out


def cat_bits_for(n_categories: int) -> int:
    """Category bits of the 3-byte word for a dialect's category count (0: none fits)."""
    return 4 if n_categories <= 16 else 5 if n_categories <= 32 else 0


def packable24(pc, cat, n_instr: int, cat_bits: int = 4) -> bool:
    """pc < n_instr <= 2^(24 - cat_bits) and categories below 2^cat_bits."""
    pc, cat = np.asarray(pc), np.asarray(cat)
    return (cat_bits in (4, 5) and n_instr <= (1 << (24 - cat_bits))
            and (pc.size == 0 or (int(pc.min()) >= 0 and int(pc.max()) < n_instr
                                  and int(cat.max()) < (1 << cat_bits))))


# streams this long bin in the one-pass hash, which reads the packed words as
# cheaply as pc / cat; shorter ones take the bucketed passes, which read pc /
# cat arrays (packing a C2-size stream cost 22 us per step, measured)
PACK_MIN_SAMPLES = 4 << 20


class DeviceSamples:
    """A raw (pc, category) stream on the device.  `packed` (default: streams
    of >= PACK_MIN_SAMPLES whose pcs fit 24 bits) stores it as one u32 word
    per sample (4 bytes instead of 5, read once by the binning); False keeps
    pc / cat arrays.  `width` 3 (packed only): the 3-byte stream of
    pack_samples24."""

    def __init__(self, pc, cat, lut, device="cuda", packed: bool | None = None, width: int | None = None):
        dev = torch.device(device)
        self.n = int(pc.shape[0])
        self.lut = to_device(np.asarray(lut, dtype=np.uint8), dev)
        if packed is None:
            packed = (int(np.asarray(pc).shape[0]) >= PACK_MIN_SAMPLES and packable(pc)
                      and not os.environ.get("LEO_NO_PACK"))
        self.packed = packed
        if width is None and packed and os.environ.get("LEO_PACK3"):
            width = 3
        self.width = 4
        cb = 4 if self.n == 0 or int(np.asarray(cat).max()) < 16 else 5
        if self.packed and width == 3 and not packable24(pc, cat, 1 << (24 - cb), cb):
            raise ValueError("DeviceSamples: the stream does not fit 3-byte words")
        if self.packed and width == 3:
            self.width = 3
            self.words = to_device(pack_samples24(pc, cat, cb), dev)
            self.pc = self.cat = None
            self.struct = abi.LeoSamples(self.n, None, None, ptr(self.lut))
            self.struct.packed = ptr(self.words)
            self.struct.packed_bytes = 3
            self.struct.packed_cat_bits = cb
        elif self.packed:
            self.words = to_device(pack_samples(pc, cat).view(np.int32), dev)
            self.pc = self.cat = None
            self.struct = abi.LeoSamples(self.n, None, None, ptr(self.lut))
            self.struct.packed = ptr(self.words)
        else:
            self.pc = to_device(np.asarray(pc, dtype=np.int32), dev)
            self.cat = to_device(np.asarray(cat, dtype=np.uint8), dev)
            self.struct = abi.LeoSamples(self.n, ptr(self.pc), ptr(self.cat), ptr(self.lut))

    @classmethod
    def from_tensors(cls, pc: torch.Tensor, cat: torch.Tensor, lut: torch.Tensor):
        self = cls.__new__(cls)
        self.n = int(pc.numel())
        self.pc, self.cat, self.lut, self.packed, self.width = pc, cat, lut, False, 4
        self.struct = abi.LeoSamples(self.n, ptr(pc), ptr(cat), ptr(lut))
        return self

    @classmethod
    def from_packed(cls, words: torch.Tensor, lut: torch.Tensor, n: int | None = None, width: int = 4,
                    cat_bits: int = 4):
        """Device u32 (int32-typed) words pc << 8 | category (width 4), or the
        3-byte stream of pack_samples24 (width 3, uint8 tensor, `n` samples)."""
        self = cls.__new__(cls)
        self.n = int(words.numel()) if n is None else int(n)
        self.words, self.lut, self.packed, self.width = words, lut, True, width
        self.pc = self.cat = None
        self.struct = abi.LeoSamples(self.n, None, None, ptr(lut))
        self.struct.packed = ptr(words)
        self.struct.packed_bytes = width
        self.struct.packed_cat_bits = cat_bits if width == 3 else 0
        return self

    def set_host_packed(self, words_host: torch.Tensor | None):
        """Pinned host words the library copies into `words` on the binning branch."""
        self.host_src = (words_host,)
        self.struct.packed_host = words_host.data_ptr() if words_host is not None else None

    def set_host_sources(self, pc_host: torch.Tensor | None, cat_host: torch.Tensor | None):
        """Pinned host tensors the library copies into pc / cat on the binning
        branch (overlapping the build); None: samples already on the device."""
        self.host_src = (pc_host, cat_host)
        self.struct.pc_host = pc_host.data_ptr() if pc_host is not None else None
        self.struct.cat_host = cat_host.data_ptr() if cat_host is not None else None


# counter slots in one int32 device vector
C_BASE, C_BASE_REG, C_PR, C_PR_REG, C_PATHS, C_DIAGS, C_BLAME, C_STATUS = range(8)


@dataclass
class Caps:
    base: int
    pruned: int
    paths: int
    diags: int
    blame: int
    scratch_scale: int = 1


class Analyzer:
    """Owns output buffers for one kernel shape; runs the fused pipeline."""

    def __init__(self, dk: DeviceKernel, device="cuda", caps: Caps | None = None,
                 debug_flags: int = 0, lines: tuple | None = None, do_slice: bool = True):
        """`lines`: optional shared (line_blame, line_stall) f64 device tensors;
        when given, this kernel accumulates into them (LEO_OPT_ACCUMULATE_LINES)
        instead of owning zero-initialised per-kernel vectors."""
        self.tracer = None
        self.debug_flags = debug_flags
        self.shared_lines = lines
        self.do_slice = do_slice
        self.ws = None                       # persistent device workspace (LeoCaps.workspace)
        self.ws_needed = C.c_int64(0)
        self.dk = dk
        self.device = torch.device(device)
        n = dk.n_instr
        nu, _ = abi.unit_counts(dk.ks)
        self.n_use_units = nu
        if caps is None:
            base = 3 * nu + 2 * n + 1024
            caps = Caps(base=base, pruned=base, paths=2 * base, diags=2 * n + 1024,
                        blame=base + n + 1024)
        self.caps = caps
        self._alloc()

    def _alloc(self):
        d, c, n = self.device, self.caps, self.dk.n_instr
        i32 = lambda m: torch.empty(max(m, 1), dtype=torch.int32, device=d)  # noqa: E731
        self.ctr = torch.zeros(8, dtype=torch.int32, device=d)
        self.b_prod, self.b_cons, self.b_meta = i32(c.base), i32(c.base), i32(c.base)
        self.p_prod, self.p_cons, self.p_meta = i32(c.pruned), i32(c.pruned), i32(c.pruned)
        self.pa_first, self.pa_np = i32(c.pruned), i32(c.pruned)
        self.pa_dist = torch.empty(max(c.pruned, 1), dtype=torch.float64, device=d)
        self.pa_len = i32(c.paths)
        self.pa_acc = torch.empty(max(c.paths, 1), dtype=torch.float64, device=d)
        self.diag = i32(6 * c.diags)
        self.bl_stalled, self.bl_edge = i32(c.blame), i32(c.blame)
        self.bl_cause, self.bl_meta = i32(c.blame), i32(c.blame)
        self.bl_sub = torch.empty(max(c.blame, 1), dtype=torch.uint8, device=d)
        self.bl_blame = torch.empty(max(c.blame, 1), dtype=torch.float64, device=d)
        self.bl_factors = torch.empty(max(4 * c.blame, 1), dtype=torch.float64, device=d)
        self.level = i32(n)
        self.bitmap = i32((n + 31) // 32)
        if self.shared_lines is not None:
            self.line_blame, self.line_stall = self.shared_lines
        else:
            self.line_blame = torch.empty(max(self.dk.n_lines, 1), dtype=torch.float64, device=d)
            self.line_stall = torch.empty(max(self.dk.n_lines, 1), dtype=torch.float64, device=d)
        cp = self.ctr.data_ptr()
        at = lambda k: cp + 4 * k  # noqa: E731
        self.s_base = abi.LeoEdges(c.base, ptr(self.b_prod), ptr(self.b_cons), ptr(self.b_meta),
                                   at(C_BASE), at(C_BASE_REG))
        self.s_pruned = abi.LeoEdges(c.pruned, ptr(self.p_prod), ptr(self.p_cons), ptr(self.p_meta),
                                     at(C_PR), at(C_PR_REG))
        self.s_paths = abi.LeoPaths(c.paths, ptr(self.pa_first), ptr(self.pa_np), ptr(self.pa_dist),
                                    ptr(self.pa_len), ptr(self.pa_acc), at(C_PATHS))
        self.s_diags = abi.LeoDiags(c.diags, ptr(self.diag), at(C_DIAGS))
        self.s_blame = abi.LeoBlame(c.blame, ptr(self.bl_stalled), ptr(self.bl_edge), ptr(self.bl_sub),
                                    ptr(self.bl_blame), ptr(self.bl_factors), at(C_BLAME),
                                    ptr(self.bl_cause), ptr(self.bl_meta))
        s = self.caps.scratch_scale
        nu, n = self.n_use_units, self.dk.n_instr
        self.s_caps = abi.LeoCaps((4 * nu + 1024) * s, (6 * nu + 1024) * s, (2 * n + 1024) * s,
                                  (n // 4 + 1024) * s, None, self.debug_flags,
                                  abi.OPT_ACCUMULATE_LINES if self.shared_lines is not None else 0,
                                  None, 0, C.pointer(self.ws_needed))
        self.status_ptr = at(C_STATUS)
        self._bind_workspace()
        self.set_tracer(self.tracer)

    def _bind_workspace(self):
        if self.ws is not None:
            self.s_caps.workspace = self.ws.data_ptr()
            self.s_caps.workspace_bytes = self.ws.numel()

    def ensure_workspace(self) -> bool:
        """Grow the persistent workspace to what the last call wanted; True if grown."""
        need = int(self.ws_needed.value)
        have = 0 if self.ws is None else self.ws.numel()
        if need <= have:
            return False
        self.ws = torch.empty(int(need * 1.25) + (1 << 20), dtype=torch.uint8, device=self.device)
        self._bind_workspace()
        return True

    def set_tracer(self, tracer: "Tracer | None"):
        self.tracer = tracer
        self.s_caps.trace = C.pointer(tracer.struct) if tracer is not None else None

    # -- launch ------------------------------------------------------------
    def launch(self, dp: DeviceProfile, cfg: abi.LeoConfig, samples: DeviceSamples | None = None,
               stream: torch.cuda.Stream | None = None, slice_: bool | None = None,
               lines: bool = True):
        st = stream or torch.cuda.current_stream(self.device)
        if slice_ is None:
            slice_ = self.do_slice
        self.ctr.zero_()
        L = lib()
        rc = L.leo_analyze(C.byref(self.dk.struct), C.byref(dp.struct),
                           C.byref(samples.struct) if samples is not None else None,
                           C.byref(cfg), C.byref(self.s_caps), C.byref(self.s_base),
                           C.byref(self.s_pruned), C.byref(self.s_paths), C.byref(self.s_diags),
                           C.byref(self.s_blame), ptr(self.bitmap) if slice_ else None,
                           ptr(self.level) if slice_ else None,
                           ptr(self.dk.line_id) if lines else None, self.dk.n_lines,
                           ptr(self.line_blame) if lines else None,
                           ptr(self.line_stall) if lines else None, self.status_ptr,
                           st.cuda_stream)
        check(rc, "leo_analyze")

    # -- CUDA graph ----------------------------------------------------------
    def capture(self, dp: DeviceProfile, cfg: abi.LeoConfig, samples: DeviceSamples | None = None,
                trace_in_graph: bool = False):
        """Capture the whole stream-ordered pipeline (no host syncs inside) into
        one CUDA graph; `replay()` then re-runs it on the current buffers.
        Buffers must already be sized (call run() first).  `trace_in_graph`:
        the tracer's events become event-record nodes of the graph (a replay
        timeline)."""
        tracer = self.tracer
        self.set_tracer(None)
        self._graph_args = (dp, cfg, samples)
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            self.launch(dp, cfg, samples)
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        if trace_in_graph and tracer is not None:
            tracer.reset()
            self.set_tracer(tracer)
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            self.launch(dp, cfg, samples)
        torch.cuda.synchronize(self.device)
        self.graph = g
        self.set_tracer(tracer)
        return g

    def replay(self):
        self.graph.replay()

    def counts(self) -> np.ndarray:
        return self.ctr.cpu().numpy()

    def run(self, dp: DeviceProfile, cfg: abi.LeoConfig, samples: DeviceSamples | None = None,
            max_retries: int = 6):
        """Launch, synchronise, grow buffers and re-run on overflow."""
        for _ in range(max_retries):
            self.launch(dp, cfg, samples)
            c = self.counts()
            status = int(np.uint32(c[C_STATUS]))
            if status & abi.ST_BAD_INPUT:
                raise ValueError("device reported malformed input (sample pc out of range or "
                                 "a block with more than two successors)")
            grow = False
            caps = self.caps
            if c[C_BASE] > caps.base or status & abi.ST_EDGE_OVERFLOW:
                caps.base = caps.pruned = int(max(c[C_BASE], caps.base) * 2) + 1024
                caps.blame = caps.base + self.dk.n_instr + 1024
                grow = True
            if c[C_PATHS] > caps.paths or status & abi.ST_PATH_OVERFLOW:
                caps.paths = int(max(c[C_PATHS], caps.paths) * 1.5) + 1024
                grow = True
            if c[C_DIAGS] > caps.diags or status & abi.ST_DIAG_OVERFLOW:
                caps.diags = int(max(c[C_DIAGS], caps.diags) * 1.5) + 1024
                grow = True
            if c[C_BLAME] > caps.blame or status & abi.ST_BLAME_OVERFLOW:
                caps.blame = int(max(c[C_BLAME], caps.blame) * 1.5) + 1024
                grow = True
            if status & abi.ST_SCRATCH_OVERFLOW:
                caps.scratch_scale *= 4
                grow = True
            if grow:
                self._alloc()
            if self.ensure_workspace():
                grow = True
            if not grow:
                return c
        raise RuntimeError("leo_analyze: buffers kept overflowing")

    # -- results -------------------------------------------------------------
    def result(self) -> dict:
        c = self.counts()
        cp = self.caps
        nb, npr = min(int(c[C_BASE]), cp.base), min(int(c[C_PR]), cp.pruned)
        npa, nd = min(int(c[C_PATHS]), cp.paths), min(int(c[C_DIAGS]), cp.diags)
        nbl = min(int(c[C_BLAME]), cp.blame)
        h = lambda t, m: t[:m].cpu().numpy()  # noqa: E731
        return dict(
            bprod=h(self.b_prod, nb), bcons=h(self.b_cons, nb),
            bmeta=h(self.b_meta, nb).view(np.uint32), n_regular=int(c[C_BASE_REG]),
            pprod=h(self.p_prod, npr), pcons=h(self.p_cons, npr),
            pmeta=h(self.p_meta, npr).view(np.uint32), p_n_regular=int(c[C_PR_REG]),
            first=h(self.pa_first, npr), npaths=h(self.pa_np, npr), pdist=h(self.pa_dist, npr),
            plen=h(self.pa_len, npa), pacc=h(self.pa_acc, npa),
            diag_records=h(self.diag, 6 * nd).reshape(-1, 6),
            e_stalled=h(self.bl_stalled, nbl), e_edge=h(self.bl_edge, nbl),
            e_cause=h(self.bl_cause, nbl), e_meta=h(self.bl_meta, nbl).view(np.uint32),
            e_sub=h(self.bl_sub, nbl), e_blame=h(self.bl_blame, nbl),
            e_factors=h(self.bl_factors, 4 * nbl).reshape(-1, 4),
            level=h(self.level, self.dk.n_instr),
            bitmap=h(self.bitmap, (self.dk.n_instr + 31) // 32).view(np.uint32),
            line_blame=h(self.line_blame, self.dk.n_lines),
            line_stall=h(self.line_stall, self.dk.n_lines),
            status=int(np.uint32(c[C_STATUS])))


    def report(self, dp: DeviceProfile, top_n: int = 10, include_unsampled: bool = False,
               chain_depth: int = 32) -> dict:
        """leo_report on the buffers of the last analysis (report assembly on
        the device: coverage, hotspot ranking, cause order, trace_chain)."""
        if not 0 <= top_n <= 4096:
            raise ValueError("top_n must be in [0, 4096] on the device report path")
        d, L = self.device, lib()
        max_causes = 16
        for _ in range(8):
            i32 = lambda m: torch.zeros(max(m, 1), dtype=torch.int32, device=d)  # noqa: E731
            cov, n_hot, hot = i32(4), i32(1), i32(top_n)
            n_causes, causes = i32(top_n), i32(top_n * max_causes)
            chain_len, chain_self = i32(top_n), i32(top_n)
            chain_node, chain_entry = i32(top_n * chain_depth), i32(top_n * chain_depth)
            status = i32(1)
            rs = abi.LeoReport(top_n, int(include_unsampled), chain_depth, max_causes, ptr(cov),
                               ptr(n_hot), ptr(hot), ptr(n_causes), ptr(causes), ptr(chain_len),
                               ptr(chain_node), ptr(chain_entry), ptr(chain_self))
            st = torch.cuda.current_stream(d)
            check(L.leo_report(C.byref(self.dk.struct), C.byref(dp.struct), C.byref(self.s_base),
                               C.byref(self.s_pruned), C.byref(self.s_blame), C.byref(rs),
                               ptr(status), st.cuda_stream), "leo_report")
            nc = n_causes.cpu().numpy()
            if int(status.item()) == 0:
                break
            max_causes = int(nc.max()) + 1
        h = lambda t: t.cpu().numpy()  # noqa: E731
        return dict(coverage=h(cov), n_hot=int(n_hot.item()), hot=h(hot), n_causes=nc,
                    causes=h(causes).reshape(max(top_n, 1), max_causes),
                    chain_len=h(chain_len), chain_node=h(chain_node).reshape(max(top_n, 1), chain_depth),
                    chain_entry=h(chain_entry).reshape(max(top_n, 1), chain_depth),
                    chain_self=h(chain_self))


def analyze_soa(ks, prof, cfg: abi.LeoConfig | None = None, samples=None, device="cuda",
                debug_flags: int = 0, packed: bool | None = None, width: int | None = None) -> dict:
    """One-shot convenience: upload, run, download."""
    dk = DeviceKernel(ks, device)
    dp = DeviceProfile(prof, ks.n_instr, device)
    ds = None
    if samples is not None:
        pc, cat, lut = samples
        ds = DeviceSamples(pc, cat, lut, device, packed=packed, width=width)
    an = Analyzer(dk, device, debug_flags=debug_flags)
    an.run(dp, cfg or abi.make_config(dialect=ks.dialect), ds)
    r = an.result()
    if ds is not None:
        r["lat"] = dp.lat.cpu().numpy()
        r["cls_cnt"] = dp.cls_cnt.cpu().numpy().reshape(-1, 8)
    return r


class Tracer:
    """Per-kernel device time of the fused pipeline (LeoTrace): CUDA events
    recorded by the library on the launching stream around each kernel (or
    only around `only_kernel`)."""

    def __init__(self, capacity: int = 4096, only_kernel: int = -1, timeline: bool = False):
        L = lib()
        self.capacity = capacity
        self.begin = (C.c_void_p * capacity)()
        self.end = (C.c_void_p * capacity)()
        self.ids = (C.c_int32 * capacity)()
        check(L.leo_events_create(capacity, self.begin), "leo_events_create")
        check(L.leo_events_create(capacity, self.end), "leo_events_create")
        self.struct = abi.LeoTrace(capacity, 0, only_kernel, 1 if timeline else 0,
                                   C.cast(self.begin, C.c_void_p),
                                   C.cast(self.end, C.c_void_p), C.cast(self.ids, C.c_void_p))

    def reset(self, only_kernel: int | None = None):
        self.struct.count = 0
        if only_kernel is not None:
            self.struct.only_kernel = only_kernel

    def records(self) -> list[tuple[str, float]]:
        """(kernel name, ms) per recorded slot; call after synchronising."""
        L = lib()
        n = min(self.struct.count, self.capacity)
        ms = (C.c_float * max(n, 1))()
        check(L.leo_events_elapsed(n, self.begin, self.end, ms), "leo_events_elapsed")
        return [(L.leo_kernel_name(self.ids[i]).decode(), float(ms[i])) for i in range(n)]

    def timeline(self) -> list[tuple[str, float, float]]:
        """(kernel name, start ms, end ms) relative to the first recorded
        launch; with timeline=True the branches keep running concurrently."""
        L = lib()
        n = min(self.struct.count, self.capacity)
        if n == 0:
            return []
        base = (C.c_void_p * n)(*([self.begin[0]] * n))
        t0 = (C.c_float * n)()
        t1 = (C.c_float * n)()
        check(L.leo_events_elapsed(n, base, self.begin, t0), "leo_events_elapsed")
        check(L.leo_events_elapsed(n, base, self.end, t1), "leo_events_elapsed")
        return [(L.leo_kernel_name(self.ids[i]).decode(), float(t0[i]), float(t1[i])) for i in range(n)]

    def summary(self) -> dict[str, float]:
        out: dict[str, float] = {}
        for name, ms in self.records():
            out[name] = out.get(name, 0.0) + ms
        return out

    def close(self):
        L = lib()
        L.leo_events_destroy(self.capacity, self.begin)
        L.leo_events_destroy(self.capacity, self.end)


def kernel_id(name: str) -> int:
    L = lib()
    i = 0
    while True:
        n = L.leo_kernel_name(i)
        if n is None:
            raise KeyError(name)
        if n.decode() == name:
            return i
        i += 1
