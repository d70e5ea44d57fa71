"""Structure-of-arrays layout of one kernel + its profile (host side, numpy).

This is the marshalling layer of the drop-in boundary: reference objects
(`KernelCfg` disasm.py:486-499, `Instruction` isa.py:215-251,
`AttachedKernel` profile.py:284-329) are flattened into the SoA arrays that
`include/leo_b200.h` declares, and device results are turned back into the
reference's `DepEdge` / `BlameEntry` objects by `api.py`.

Encoding rules
  * operand records per instruction, in the order the reference iterates them
    (`per_use_link` depgraph.py:212-217): srcs, then the guard, then dests;
  * register units (depgraph.py:41) get dense ids `unit_base[class] + index`;
  * sync variants (isa.py:153-206) pack into two u32 words (see the header);
  * profile accessors (profile.py:304-329) become dense per-instruction arrays;
    the vendor->common stall map (profile.py:106-111) is applied here, so the
    device sees `cls_cnt[N, 8]`.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import enums as E

UNKNOWN_LINE = "<unknown>"


@dataclass
class KernelSoA:
    name: str
    dialect: str
    opclass: np.ndarray          # u8[N]
    block_of: np.ndarray         # i32[N]
    opnd_ptr: np.ndarray         # i32[N+1]
    opnd: np.ndarray             # u32[M]
    sync_kind: np.ndarray        # u8[N]
    sync_a: np.ndarray           # u32[N]
    sync_b: np.ndarray           # u32[N]
    blk_first: np.ndarray        # i32[B]
    blk_last: np.ndarray         # i32[B]
    succ_ptr: np.ndarray         # i32[B+1]
    succ: np.ndarray             # i32[*]
    pred_ptr: np.ndarray         # i32[B+1]
    pred: np.ndarray             # i32[*]
    unit_base: np.ndarray        # i32[8]
    n_units: int
    offset: np.ndarray           # i64[N]   host only (diagnostic text)
    line_id: np.ndarray          # i32[N]   index into `lines`
    lines: list = field(default_factory=list)       # line key strings
    prefix_diagnostics: tuple = ()                  # attach + cfg diagnostics
    seg_block: np.ndarray | None = None             # batches: members' first blocks [S+1]

    @property
    def n_instr(self) -> int:
        return int(self.opclass.shape[0])

    @property
    def n_blocks(self) -> int:
        return int(self.blk_first.shape[0])

    @property
    def dialect_idx(self) -> int:
        return E.DIALECT_IDX[self.dialect]


@dataclass
class ProfileSoA:
    period: int
    lat: np.ndarray              # i32[N]
    cls_cnt: np.ndarray          # i32[N, 8]
    exec_cnt: np.ndarray         # i64[N]  (-1 = None)
    total: np.ndarray            # i32[N]  (-1 = None)
    eff: np.ndarray              # f64[N]
    sampled: np.ndarray          # u8[N]


def pack_opnd(role: int, rc: int, index: int, span: int) -> int:
    if not (0 <= index < 65536 and 1 <= span < 256):
        raise ValueError(f"register index/span out of SoA range: {index}/{span}")
    return index | (span << 16) | (rc << 24) | (role << 27)


def opnd_fields(rec):
    rec = np.asarray(rec, dtype=np.uint32)
    return (rec >> 27) & 3, (rec >> 24) & 7, rec & 0xFFFF, (rec >> 16) & 0xFF


def line_key(src_loc) -> str:
    """Per-source-line rollup key: the SourceLoc head `file:line`
    (isa.py:141-150); instructions without a location map to <unknown>."""
    if src_loc is None:
        return UNKNOWN_LINE
    return f"{src_loc.file}:{src_loc.line}"


# ---------------------------------------------------------------------------
# reference objects -> SoA

def encode_cfg(cfg, line_table: dict | None = None) -> KernelSoA:
    """Flatten a reference `KernelCfg` (duck-typed) into a KernelSoA."""
    instrs = cfg.instructions
    n = len(instrs)
    dialect = cfg.dialect.value
    ext = [0] * 8
    ops: list[int] = []
    ptr = np.zeros(n + 1, dtype=np.int32)
    opclass = np.zeros(n, dtype=np.uint8)
    sync_kind = np.zeros(n, dtype=np.uint8)
    sync_a = np.full(n, E.NONE_U32, dtype=np.uint32)
    sync_b = np.full(n, E.NONE_U32, dtype=np.uint32)
    offset = np.zeros(n, dtype=np.int64)
    line_id = np.zeros(n, dtype=np.int32)
    if line_table is None:
        line_table = {}
    for i, ins in enumerate(instrs):
        opclass[i] = E.OC_IDX[ins.opcode_class.value]
        offset[i] = ins.offset
        for role, refs in ((E.ROLE_SRC, ins.srcs),
                           (E.ROLE_GUARD, (ins.guard.register,) if ins.guard is not None else ()),
                           (E.ROLE_DST, ins.dests)):
            for ref in refs:
                rc = E.RC_IDX[ref.reg_class.value]
                ops.append(pack_opnd(role, rc, ref.index, ref.span))
                ext[rc] = max(ext[rc], ref.index + ref.span)
        ptr[i + 1] = len(ops)
        s = ins.sync
        if s is not None:
            tname = type(s).__name__
            if tname == "Waitcnt":
                sync_kind[i] = E.SYNC_WAITCNT
                sync_a[i] = E.NONE_U32 if s.vmcnt is None else s.vmcnt
                sync_b[i] = E.NONE_U32 if s.lgkmcnt is None else s.lgkmcnt
            elif tname == "BarrierCtl":
                sync_kind[i] = E.SYNC_BARRIER
                w = sum(1 << b for b in s.write_set)
                r = sum(1 << b for b in s.read_set)
                wt = sum(1 << b for b in s.wait_mask)
                sync_a[i] = w | (r << 8) | (wt << 16)
                sync_b[i] = E.NONE_U32 if s.issue_stall_cycles is None else s.issue_stall_cycles
            elif tname == "Swsb":
                sync_kind[i] = E.SYNC_SWSB
                sync_a[i] = E.NONE_U32 if s.set_token is None else s.set_token
                sync_b[i] = sum(1 << t for t in (set(s.wait_dst) | set(s.wait_src)))
            else:
                raise TypeError(f"unknown sync info {tname}")
        key = line_key(ins.src_loc)
        lid = line_table.get(key)
        if lid is None:
            lid = line_table[key] = len(line_table)
        line_id[i] = lid
    unit_base = np.zeros(8, dtype=np.int32)
    acc = 0
    for c in range(8):
        unit_base[c] = acc
        acc += ext[c]
    blocks = cfg.blocks
    nb = len(blocks)
    blk_first = np.array([b.first_index for b in blocks], dtype=np.int32)
    blk_last = np.array([b.last_index for b in blocks], dtype=np.int32)
    succ_ptr = np.zeros(nb + 1, dtype=np.int32)
    pred_ptr = np.zeros(nb + 1, dtype=np.int32)
    succ, pred = [], []
    for b in blocks:
        succ.extend(b.succs)
        pred.extend(b.preds)
        succ_ptr[b.id + 1] = len(succ)
        pred_ptr[b.id + 1] = len(pred)
    lines = [None] * len(line_table)
    for k, v in line_table.items():
        lines[v] = k
    return KernelSoA(
        name=cfg.kernel_name, dialect=dialect, opclass=opclass,
        block_of=np.asarray(cfg.block_of, dtype=np.int32),
        opnd_ptr=ptr, opnd=np.asarray(ops, dtype=np.uint32),
        sync_kind=sync_kind, sync_a=sync_a, sync_b=sync_b,
        blk_first=blk_first, blk_last=blk_last,
        succ_ptr=succ_ptr, succ=np.asarray(succ, dtype=np.int32),
        pred_ptr=pred_ptr, pred=np.asarray(pred, dtype=np.int32),
        unit_base=unit_base, n_units=int(acc), offset=offset, line_id=line_id,
        lines=lines, prefix_diagnostics=tuple(cfg.diagnostics))


def encode_profile(attached) -> ProfileSoA:
    """Dense per-instruction arrays equal to the AttachedKernel accessors
    (profile.py:304-329)."""
    cfg = attached.cfg
    dialect = cfg.dialect.value
    smap = E.STALL_MAPS[dialect]
    n = len(cfg.instructions)
    lat = np.zeros(n, dtype=np.int32)
    cls = np.zeros((n, 8), dtype=np.int32)
    exec_cnt = np.full(n, -1, dtype=np.int64)
    total = np.full(n, -1, dtype=np.int32)
    eff = np.ones(n, dtype=np.float64)
    sampled = np.zeros(n, dtype=np.uint8)
    for i, rec in enumerate(attached.samples):
        lat[i] = rec.latency_samples
        for cat, cnt in rec.vendor_counts:
            cls[i, E.CS_IDX[smap[E.norm_category(cat)]]] += cnt
        if rec.exec_count is not None:
            exec_cnt[i] = rec.exec_count
        if rec.total_samples is not None:
            total[i] = rec.total_samples
        eff[i] = rec.efficiency
        sampled[i] = 1 if attached.sampled[i] else 0
    return ProfileSoA(period=int(attached.period), lat=lat, cls_cnt=cls, exec_cnt=exec_cnt,
                      total=total, eff=eff, sampled=sampled)


def encode_attached(attached, line_table: dict | None = None):
    ks = encode_cfg(attached.cfg, line_table)
    ks.prefix_diagnostics = tuple(attached.diagnostics) + tuple(attached.cfg.diagnostics)
    return ks, encode_profile(attached)


# ---------------------------------------------------------------------------
# SoA -> reference objects (used by tests to run the reference on synthetic
# SoA inputs, and by api.py to rebuild DepEdge/RegisterRef values)

_PLACEHOLDER_MNEMONIC = "op"


def decode_to_reference(ks: KernelSoA, prof: ProfileSoA | None = None, st=None):
    """Rebuild reference `KernelCfg` (+ `AttachedKernel`) objects from SoA.

    `st` is the imported `stalltrace` package.  Mnemonics are placeholders:
    the analysis never re-classifies (it reads `opcode_class`)."""
    isa, disasm, profile = st.isa, st.disasm, st.profile
    dialect = isa.Dialect(ks.dialect)
    rcs = [isa.RegClass(v) for v in E.REG_CLASSES]
    ocs = [isa.OpcodeClass(v) for v in E.OPCODE_CLASSES]
    instrs = []
    role, rc, idx, span = opnd_fields(ks.opnd)
    for i in range(ks.n_instr):
        srcs, dests, guard = [], [], None
        for k in range(ks.opnd_ptr[i], ks.opnd_ptr[i + 1]):
            ref = isa.RegisterRef(rcs[int(rc[k])], int(idx[k]), int(span[k]))
            if role[k] == E.ROLE_SRC:
                srcs.append(ref)
            elif role[k] == E.ROLE_GUARD:
                guard = isa.Guard(ref)
            else:
                dests.append(ref)
        sk = int(ks.sync_kind[i])
        a, b = int(ks.sync_a[i]), int(ks.sync_b[i])
        sync = None
        if sk == E.SYNC_WAITCNT:
            sync = isa.Waitcnt(vmcnt=None if a == E.NONE_U32 else a,
                               lgkmcnt=None if b == E.NONE_U32 else b)
        elif sk == E.SYNC_BARRIER:
            bits = lambda m: frozenset(x for x in range(1, 7) if m >> x & 1)
            sync = isa.BarrierCtl(write_set=bits(a & 0xFF), read_set=bits((a >> 8) & 0xFF),
                                  wait_mask=bits((a >> 16) & 0xFF),
                                  issue_stall_cycles=None if b == E.NONE_U32 else b)
        elif sk == E.SYNC_SWSB:
            sync = isa.Swsb(set_token=None if a == E.NONE_U32 else a,
                            wait_dst=frozenset(t for t in range(32) if b >> t & 1))
        key = ks.lines[ks.line_id[i]] if ks.lines else UNKNOWN_LINE
        loc = None
        if key != UNKNOWN_LINE:
            f, ln = key.rsplit(":", 1)
            loc = isa.SourceLoc(f, int(ln))
        instrs.append(isa.Instruction(
            offset=int(ks.offset[i]), dialect=dialect, mnemonic=_PLACEHOLDER_MNEMONIC,
            opcode_class=ocs[int(ks.opclass[i])], dests=tuple(dests), srcs=tuple(srcs),
            guard=guard, sync=sync, src_loc=loc))
    blocks = []
    for b in range(ks.n_blocks):
        blocks.append(disasm.BasicBlock(
            id=b, first_index=int(ks.blk_first[b]), last_index=int(ks.blk_last[b]),
            succs=tuple(int(x) for x in ks.succ[ks.succ_ptr[b]:ks.succ_ptr[b + 1]]),
            preds=tuple(int(x) for x in ks.pred[ks.pred_ptr[b]:ks.pred_ptr[b + 1]])))
    cfg = disasm.KernelCfg(
        kernel_name=ks.name, dialect=dialect, instructions=tuple(instrs),
        blocks=tuple(blocks), entry=0, labels={}, unreachable=frozenset(),
        diagnostics=(), block_of=tuple(int(x) for x in ks.block_of))
    if prof is None:
        return cfg
    cats = E.vendor_categories(ks.dialect)
    # one representative vendor category per common class
    rep = {}
    for c in cats:
        rep.setdefault(E.CS_IDX[E.STALL_MAPS[ks.dialect][c]], c)
    samples = []
    sampled = []
    for i in range(ks.n_instr):
        if not prof.sampled[i]:
            samples.append(profile.InstructionSamples(offset=0, vendor_counts=(), latency_samples=0))
            sampled.append(False)
            continue
        vc = tuple((rep[c], int(prof.cls_cnt[i, c])) for c in range(8) if prof.cls_cnt[i, c] > 0)
        samples.append(profile.InstructionSamples(
            offset=int(ks.offset[i]), vendor_counts=vc, latency_samples=int(prof.lat[i]),
            total_samples=None if prof.total[i] < 0 else int(prof.total[i]),
            exec_count=None if prof.exec_cnt[i] < 0 else int(prof.exec_cnt[i]),
            efficiency=float(prof.eff[i])))
        sampled.append(True)
    kp = profile.KernelProfile(kernel_name=ks.name, dialect=dialect,
                               sampling_period_cycles=int(prof.period),
                               samples=tuple(s for s, f in zip(samples, sampled) if f))
    att = profile.AttachedKernel(cfg=cfg, profile=kp, samples=tuple(samples),
                                 sampled=tuple(sampled), skid_offsets=(), diagnostics=())
    return att
