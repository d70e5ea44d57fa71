"""Seeded synthetic workloads of the shapes BASELINE.json names.

Produces `KernelSoA` + `ProfileSoA` + a raw PC-sample stream directly (numpy,
PCG64), so they run on the GPU box where the reference is absent.  Shapes:

  C2  amd    N=10,000   S=1M     loops <=3 deep, diamonds, s_waitcnt 12 %
  C3  intel  N=50,000   S=5M     `while` nests <=8 deep, goto skips, SWSB tokens
  C4  2,000 kernels x 20,000, vendor [nvidia, amd, intel][k % 3], S=100k each
  C5  nvidia N=1,000,000 S=100M  branchy, barrier masks + stall cycles

PCs follow Zipf(1.1) over a seed-permuted instruction order; the vendor
category of a sample comes from a class-dependent mix (loads and waits 80 %
memory).  Every instruction carries exec_count in [256, 4096]; efficiency is
1.0 except 10 % of memory operations at U(0.1, 1.0) rounded to 3 decimals
(generators.py:187); period 100.  Source lines come from a shared pool of
files so that per-line totals overlap across kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import enums as E
from .soa import KernelSoA, ProfileSoA, pack_opnd

OC = E.OC_IDX
RC = E.RC_IDX


class LineTable:
    """Pool of `n_files` files with U(100, 2000) lines each; global line id =
    file base + line - 1; the last id is `<unknown>`."""

    def __init__(self, n_files: int, seed: int = 12345):
        rng = np.random.Generator(np.random.PCG64(seed))
        self.sizes = rng.integers(100, 2001, size=n_files).astype(np.int64)
        self.base = np.concatenate([[0], np.cumsum(self.sizes)])
        self.n = int(self.base[-1]) + 1

    def __len__(self):
        return self.n

    def __iter__(self):
        return (self[i] for i in range(self.n))

    def __getitem__(self, lid: int) -> str:
        lid = int(lid)
        if lid < 0 or lid >= self.n:
            raise IndexError(lid)
        if lid == self.n - 1:
            return "<unknown>"
        f = int(np.searchsorted(self.base, lid, side="right") - 1)
        return f"src/file{f:04d}.cpp:{lid - int(self.base[f]) + 1}"


@dataclass
class Workload:
    kernel: KernelSoA
    profile: ProfileSoA          # metadata (exec/total/eff/sampled); lat/cls from binning
    pc: np.ndarray               # i32[S]
    cat: np.ndarray              # u8[S]
    lut: np.ndarray              # u8[256] vendor category -> CommonStall

    @property
    def n_samples(self) -> int:
        return int(self.pc.shape[0])


# ---------------------------------------------------------------------------
# opcode mixes: (opclass, probability, has_dest)

_MIX = {
    "amd": [("global_load", .08), ("global_store", .04), ("local_load", .03),
            ("scalar_load", .03), ("local_store", .02), ("sync_wait", .12),
            ("fp_arith", .28), ("int_arith", .27), ("conversion", .05), ("other", .08)],
    "nvidia": [("global_load", .10), ("global_store", .03), ("local_load", .03),
               ("fp_arith", .30), ("int_arith", .38), ("conversion", .04), ("other", .10),
               ("barrier_all", .02)],
    "intel": [("send", .12), ("fp_arith", .35), ("int_arith", .33), ("conversion", .05),
              ("other", .15)],
}
_NO_DEST = {OC["global_store"], OC["local_store"], OC["control_flow"], OC["sync_wait"],
            OC["barrier_all"], OC["nop"]}

_SHAPE = {
    #          mean block, loop depth, p_open, p_close, p_diamond, n vregs, n sregs
    "amd": dict(blk=10, depth=3, p_open=.06, p_close=.10, p_fwd=.15, nv=128, ns=64),
    "nvidia": dict(blk=20, depth=3, p_open=.05, p_close=.12, p_fwd=.25, nv=64, ns=0),
    "intel": dict(blk=10, depth=8, p_open=.10, p_close=.16, p_fwd=.10, nv=48, ns=0),
}


def _cfg(rng, n_instr: int, dialect: str):
    """Block sizes + terminators: nested loops (backward conditional branch to
    the loop header), forward conditional skips, exit at the end."""
    sh = _SHAPE[dialect]
    sizes = []
    left = n_instr
    while left > 0:
        s = int(min(left, max(2, rng.poisson(sh["blk"] - 2) + 2)))
        if 0 < left - s < 2:
            s = left
        sizes.append(s)
        left -= s
    nb = len(sizes)
    target = np.full(nb, -1, dtype=np.int64)     # -1 fallthrough, -2 exit
    stack: list[int] = []
    u = rng.random((nb, 4))
    for b in range(nb - 1):
        if len(stack) < sh["depth"] and u[b, 0] < sh["p_open"]:
            stack.append(b)
        if stack and stack[-1] < b and u[b, 1] < sh["p_close"]:
            target[b] = stack.pop()              # latch -> header
        elif u[b, 2] < sh["p_fwd"] and b + 2 < nb:
            target[b] = b + 2 + int(u[b, 3] * 2)  # skip 1-2 blocks
            target[b] = min(target[b], nb - 1)
    target[nb - 1] = -2
    return np.asarray(sizes, dtype=np.int64), target


def make_kernel(dialect: str, n_instr: int, seed: int, name: str | None = None,
                lines: LineTable | None = None) -> tuple[KernelSoA, ProfileSoA]:
    rng = np.random.Generator(np.random.PCG64(seed))
    sizes, target = _cfg(rng, n_instr, dialect)
    nb = sizes.shape[0]
    n = int(sizes.sum())
    blk_first = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int32)
    blk_last = (blk_first + sizes - 1).astype(np.int32)
    block_of = np.repeat(np.arange(nb, dtype=np.int32), sizes)

    # successors [target, fallthrough] (disasm.py:572), preds sorted (:596)
    succ_lists = []
    for b in range(nb):
        t = int(target[b])
        if t == -2:
            succ_lists.append([])
        elif t == -1:
            succ_lists.append([b + 1])
        else:
            succ_lists.append([t] if t == b + 1 else [t, b + 1])
    succ_ptr = np.zeros(nb + 1, dtype=np.int32)
    succ_ptr[1:] = np.cumsum([len(s) for s in succ_lists])
    succ = np.asarray([x for s in succ_lists for x in s], dtype=np.int32)
    pred_lists = [[] for _ in range(nb)]
    for b, s in enumerate(succ_lists):
        for x in s:
            pred_lists[x].append(b)
    pred_ptr = np.zeros(nb + 1, dtype=np.int32)
    pred_ptr[1:] = np.cumsum([len(p) for p in pred_lists])
    pred = np.asarray([x for p in pred_lists for x in sorted(p)], dtype=np.int32)

    # opcode classes
    names, probs = zip(*_MIX[dialect])
    probs = np.asarray(probs) / np.sum(probs)
    opclass = np.asarray([OC[c] for c in names], dtype=np.uint8)[rng.choice(len(names), size=n, p=probs)]
    is_branch = np.zeros(n, dtype=bool)
    is_branch[blk_last[target != -1]] = True
    opclass[is_branch] = OC["control_flow"]
    opclass[blk_last[target == -2]] = OC["control_flow"]
    # the first instructions define predicates used by the branch guards
    pred_def = (rng.random(n) < 0.03) & (opclass == OC["int_arith"])

    sh = _SHAPE[dialect]
    nv, ns = sh["nv"], sh["ns"]
    has_dest = ~np.isin(opclass, list(_NO_DEST))
    r = rng.random((n, 8))
    span_of = lambda x: np.where(x < .75, 1, np.where(x < .95, 2, 4))  # noqa: E731
    if dialect == "nvidia":
        span_of = lambda x: np.where(x < .85, 1, 2)  # noqa: E731
    dspan = span_of(r[:, 0])
    didx = (r[:, 1] * (nv - dspan)).astype(np.int64)
    drc = np.full(n, RC["vector_gpr"], dtype=np.int64)
    if ns:
        sdst = (opclass == OC["scalar_load"]) | ((opclass == OC["int_arith"]) & (r[:, 2] < .3))
        drc[sdst] = RC["scalar_gpr"]
        didx[sdst] = (r[sdst, 1] * (ns - dspan[sdst])).astype(np.int64)
    n_src = np.where(r[:, 3] < .35, 1, 2)
    n_src[opclass == OC["sync_wait"]] = 0
    n_src[opclass == OC["barrier_all"]] = 0
    n_src[is_branch] = 0
    n_src[blk_last[target == -2]] = 0
    sspan = span_of(rng.random((n, 2)))
    sidx = (rng.random((n, 2)) * (nv - sspan)).astype(np.int64)
    src_scalar = rng.random((n, 2)) < (0.25 if ns else 0.0)
    guard = np.full(n, -1, dtype=np.int64)
    guard[is_branch] = rng.integers(0, 2, size=int(is_branch.sum()))
    gmask = (rng.random(n) < 0.04) & ~is_branch
    guard[gmask] = rng.integers(0, 2, size=int(gmask.sum()))

    # sync words
    sync_kind = np.zeros(n, dtype=np.uint8)
    sync_a = np.full(n, E.NONE_U32, dtype=np.uint32)
    sync_b = np.full(n, E.NONE_U32, dtype=np.uint32)
    if dialect == "amd":
        w = opclass == OC["sync_wait"]
        sync_kind[w] = E.SYNC_WAITCNT
        k = int(w.sum())
        vm = rng.choice([0, 1, 2, 3], size=k, p=[.6, .15, .15, .10]).astype(np.uint32)
        has_vm = rng.random(k) < .85
        has_lg = rng.random(k) < .30
        has_vm |= ~has_lg
        sync_a[w] = np.where(has_vm, vm, E.NONE_U32)
        sync_b[w] = np.where(has_lg, 0, E.NONE_U32)
    elif dialect == "nvidia":
        sync_kind[:] = E.SYNC_BARRIER
        loads = np.isin(opclass, [OC["global_load"], OC["local_load"]])
        wbar = rng.integers(1, 7, size=n)
        a = np.where(loads, 1 << wbar, 0).astype(np.uint32)
        waits = (rng.random(n) < .10) & ~loads
        wait_bar = rng.integers(1, 7, size=n)
        a |= np.where(waits, (1 << wait_bar) << 16, 0).astype(np.uint32)
        sync_a[:] = a
        stall = rng.choice([0, 1, 2, 4, 6], size=n, p=[.05, .45, .25, .15, .10])
        sync_b[:] = stall.astype(np.uint32)
    else:  # intel
        sends = np.flatnonzero(opclass == OC["send"])
        sync_kind[sends] = E.SYNC_SWSB
        sync_a[sends] = (np.arange(sends.shape[0]) % 32).astype(np.uint32)
        sync_b[sends] = 0
        # ~20 % of ALU ops wait sbid.wait.dst, 5 % sbid.wait.src,
        # on a token set within the last 16 instructions in layout order -- in
        # the waiter's block or in an earlier one (cross-block setter searches
        # over the nested loops).  The SoA keeps dst | src as one mask
        # (depgraph.py:466-482 waits on their union).
        alu = np.isin(opclass, [OC["fp_arith"], OC["int_arith"], OC["conversion"]])
        u = rng.random(n)
        for lo, hi in ((0.0, 0.20), (0.20, 0.25)):          # dst, then src waits
            cand = np.flatnonzero(alu & (u >= lo) & (u < hi))
            back = rng.integers(1, 17, size=cand.shape[0])   # setter 1..16 instructions back
            pos = np.searchsorted(sends, cand - back, side="right") - 1
            ok = (pos >= 0)
            cand, pos = cand[ok], pos[ok]
            ok = (cand - sends[pos]) <= 16
            cand, pos = cand[ok], pos[ok]
            sync_kind[cand] = E.SYNC_SWSB                    # (sync_a stays None: no set)
            sync_b[cand] = np.where(sync_b[cand] == E.NONE_U32, 0, sync_b[cand]) | \
                (np.uint32(1) << sync_a[sends[pos]]).astype(np.uint32)

    # operand CSR: srcs, guard, dests
    cnt = n_src + (guard >= 0) + has_dest
    opnd_ptr = np.zeros(n + 1, dtype=np.int32)
    opnd_ptr[1:] = np.cumsum(cnt)
    m = int(opnd_ptr[-1])
    opnd = np.zeros(m, dtype=np.uint32)
    pos = opnd_ptr[:-1].astype(np.int64).copy()

    def put(mask, role, rc, idx, span):
        sel = np.flatnonzero(mask)
        rcv = np.broadcast_to(rc, (n,))[sel] if np.ndim(rc) else np.full(sel.shape, rc)
        vals = (idx[sel].astype(np.uint32) | (span[sel].astype(np.uint32) << 16)
                | (rcv.astype(np.uint32) << 24) | np.uint32(role << 27))
        opnd[pos[sel]] = vals
        pos[sel] += 1

    for s in range(2):
        msk = n_src > s
        rcs = np.where(src_scalar[:, s], RC["scalar_gpr"], RC["vector_gpr"])
        idx = np.where(src_scalar[:, s], sidx[:, s] % np.maximum(ns - sspan[:, s], 1), sidx[:, s]) if ns else sidx[:, s]
        put(msk, E.ROLE_SRC, rcs, idx, sspan[:, s])
    one = np.ones(n, dtype=np.int64)
    put(guard >= 0, E.ROLE_GUARD, RC["predicate"], np.maximum(guard, 0), one)
    put(has_dest & ~pred_def, E.ROLE_DST, drc, didx, dspan)
    put(pred_def, E.ROLE_DST, RC["predicate"], rng.integers(0, 2, size=n), one)
    assert np.array_equal(pos, opnd_ptr[1:])

    ext = np.zeros(8, dtype=np.int64)
    rcv = (opnd >> 24) & 7
    top = (opnd & 0xFFFF) + ((opnd >> 16) & 0xFF)
    for c in range(8):
        sel = rcv == c
        if sel.any():
            ext[c] = int(top[sel].max())
    unit_base = np.concatenate([[0], np.cumsum(ext)[:-1]]).astype(np.int32)

    # source lines: runs of instructions share a line; regions of 64 share a file
    if lines is None:
        lines = LineTable(64, seed=999)
    nf = lines.sizes.shape[0]
    region = np.arange(n) // 64
    nreg = int(region.max()) + 1
    rfile = rng.integers(0, nf, size=nreg)
    rstart = (rng.random(nreg) * lines.sizes[rfile]).astype(np.int64)
    ln = np.minimum(rstart[region] + (np.arange(n) % 64) // 4, lines.sizes[rfile[region]] - 1)
    line_id = (lines.base[rfile[region]] + ln).astype(np.int32)
    line_id[rng.random(n) < .02] = lines.n - 1

    offset = np.arange(n, dtype=np.int64) * (4 if dialect == "amd" else 16)
    ks = KernelSoA(
        name=name or f"{dialect}_{n}_{seed}", dialect=dialect, opclass=opclass,
        block_of=block_of, opnd_ptr=opnd_ptr, opnd=opnd, sync_kind=sync_kind,
        sync_a=sync_a, sync_b=sync_b, blk_first=blk_first, blk_last=blk_last,
        succ_ptr=succ_ptr, succ=succ, pred_ptr=pred_ptr, pred=pred,
        unit_base=np.concatenate([unit_base, np.zeros(0, np.int32)]).astype(np.int32),
        n_units=int(ext.sum()), offset=offset, line_id=line_id, lines=lines)

    mem = np.isin(opclass, list(E.MEMORY_CLASSES))
    eff = np.ones(n, dtype=np.float64)
    low = mem & (rng.random(n) < .10)
    eff[low] = np.round(rng.uniform(0.1, 1.0, size=int(low.sum())), 3)
    prof = ProfileSoA(
        period=100, lat=np.zeros(n, np.int32), cls_cnt=np.zeros((n, 8), np.int32),
        exec_cnt=rng.integers(256, 4097, size=n).astype(np.int64),
        total=np.full(n, -1, dtype=np.int32), eff=eff, sampled=np.ones(n, dtype=np.uint8))
    return ks, prof


def _category_of_class(dialect: str):
    """Primary vendor category id per OpcodeClass."""
    cats = E.vendor_categories(dialect)
    mem = {"nvidia": "memory dependency", "amd": "waiting for memory",
           "intel": "memory send operations"}[dialect]
    exe = {"nvidia": "execution dependency", "amd": "alu dependency",
           "intel": "pipeline hazards"}[dialect]
    other = {"nvidia": "pipe busy", "amd": "pipeline stall", "intel": "distribution stalls"}[dialect]
    sync = {"nvidia": "synchronization", "amd": "barrier wait", "intel": "sbidstall"}[dialect]
    prim = np.full(16, cats.index(other), dtype=np.uint8)
    for c in ("global_load", "local_load", "scalar_load", "constant_load", "atomic", "send",
              "global_store", "local_store", "sync_wait"):
        prim[OC[c]] = cats.index(mem)
    for c in ("fp_arith", "int_arith", "conversion"):
        prim[OC[c]] = cats.index(exe)
    prim[OC["barrier_all"]] = cats.index(sync)
    return prim, len(cats)


def make_samples(ks: KernelSoA, n_samples: int, seed: int, chunk: int = 1 << 24):
    """Raw (pc, category) stream: PC ~ Zipf(1.1) over a permuted order."""
    rng = np.random.Generator(np.random.PCG64(seed ^ 0x5A5A))
    n = ks.n_instr
    perm = rng.permutation(n).astype(np.int32)
    w = np.arange(1, n + 1, dtype=np.float64) ** -1.1
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    prim, ncat = _category_of_class(ks.dialect)
    prim_i = prim[ks.opclass]
    pc = np.empty(n_samples, dtype=np.int32)
    cat = np.empty(n_samples, dtype=np.uint8)
    for s0 in range(0, n_samples, chunk):
        s1 = min(n_samples, s0 + chunk)
        u = rng.random(s1 - s0)
        rank = np.minimum(np.searchsorted(cdf, u, side="right"), n - 1)
        p = perm[rank]
        pc[s0:s1] = p
        alt = rng.integers(0, ncat, size=s1 - s0).astype(np.uint8)
        cat[s0:s1] = np.where(rng.random(s1 - s0) < 0.8, prim_i[p], alt)
    return pc, cat


def make_workload(dialect: str, n_instr: int, n_samples: int, seed: int,
                  lines: LineTable | None = None, name: str | None = None) -> Workload:
    ks, prof = make_kernel(dialect, n_instr, seed, name=name, lines=lines)
    pc, cat = make_samples(ks, n_samples, seed)
    return Workload(kernel=ks, profile=prof, pc=pc, cat=cat, lut=E.category_lut(dialect))


def bin_host(wl: Workload) -> ProfileSoA:
    """numpy.bincount binning of the raw stream into a full ProfileSoA (for
    tests and the CPU baseline; the product bins on the device)."""
    n = wl.kernel.n_instr
    cs = wl.lut[wl.cat].astype(np.int64)
    cls = np.bincount(wl.pc.astype(np.int64) * 8 + cs, minlength=n * 8).astype(np.int32).reshape(n, 8)
    p = wl.profile
    return ProfileSoA(period=p.period, lat=cls.sum(axis=1).astype(np.int32), cls_cnt=cls,
                      exec_cnt=p.exec_cnt, total=p.total, eff=p.eff, sampled=p.sampled)


# ---------------------------------------------------------------------------
# the five configs (BASELINE.json "configs")

CONFIGS = {
    "c2": dict(dialect="amd", n_instr=10_000, n_samples=1_000_000, seed=2, files=64),
    "c3": dict(dialect="intel", n_instr=50_000, n_samples=5_000_000, seed=3, files=256),
    "c5": dict(dialect="nvidia", n_instr=1_000_000, n_samples=100_000_000, seed=5, files=4096),
}
C4_KERNELS, C4_INSTR, C4_SAMPLES = 2000, 20_000, 100_000


def config_workload(tag: str, scale: float = 1.0, seed_offset: int = 0) -> Workload:
    c = CONFIGS[tag]
    lines = LineTable(c["files"], seed=999)
    return make_workload(c["dialect"], max(64, int(c["n_instr"] * scale)),
                         max(1, int(c["n_samples"] * scale)), c["seed"] + seed_offset,
                         lines=lines, name=f"{tag}_{c['seed'] + seed_offset}")


def c4_kernel(k: int, lines: LineTable, scale: float = 1.0) -> Workload:
    dialect = E.DIALECTS[k % 3]
    return make_workload(dialect, max(64, int(C4_INSTR * scale)), max(1, int(C4_SAMPLES * scale)),
                         40_000 + k, lines=lines, name=f"c4_{k}")
