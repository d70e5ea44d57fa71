"""Binary raw PC-sample stream.

The reference reads pre-binned, aggregated JSON profiles (profile.py:186-263;
pkg/README.md:96-116).  At 100 M samples a text format cannot feed stage-0
binning, so raw samples travel as a flat binary file that maps straight into
the arrays `LeoSamples` wants: the file is memory-mapped, copied once into
pinned memory and from there by the library's binning branch.

Layout (little-endian, sections 16-byte aligned):

    magic     8 B   b"LEOSMP01"
    n_samples u64
    n_instr   u32   instructions of the kernel the pcs index
    period    u32   sampling period in cycles (profile.py:122)
    dialect   u32   index into enums.DIALECTS
    n_cat     u32   vendor categories listed below
    name_len  u32   kernel name bytes
    cat_len   u32   category table bytes ('\\n'-joined, normalised names)
    name, categories, pad16
    pc        i32[n_samples]   instruction index
    pad16
    cat       u8[n_samples]    index into the file's category table

Category ids are the file's own: the reader maps each name to a CommonStall
through the dialect's stall map (profile.py:52-111) and builds the uint8
`cat_to_cs` table, so producers need not know this package's id order.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import enums as E

MAGIC = b"LEOSMP01"
_HDR = struct.Struct("<8sQIIIIII")


def _pad16(n: int) -> int:
    return (n + 15) & ~15


@dataclass
class RawSamples:
    kernel_name: str
    dialect: str
    period: int
    n_instr: int
    categories: tuple
    pc: np.ndarray          # i32[S] (memory-mapped when read from a file)
    cat: np.ndarray         # u8[S]

    @property
    def n_samples(self) -> int:
        return int(self.pc.shape[0])

    def lut(self) -> np.ndarray:
        """uint8[256] file category id -> CommonStall index (map_stall,
        profile.py:106-111; unknown names map to `other`)."""
        lut = np.full(256, E.CS_IDX["other"], dtype=np.uint8)
        m = E.STALL_MAPS[self.dialect]
        for i, name in enumerate(self.categories):
            lut[i] = E.CS_IDX[m.get(E.norm_category(name), "other")]
        return lut


def write(path, rs: RawSamples) -> int:
    """Write `rs`; returns the file size."""
    pc = np.ascontiguousarray(rs.pc, dtype=np.int32)
    cat = np.ascontiguousarray(rs.cat, dtype=np.uint8)
    if pc.shape != cat.shape:
        raise ValueError("pc and cat must have the same length")
    if len(rs.categories) > 256:
        raise ValueError("at most 256 vendor categories")
    if pc.size and (pc.min() < 0 or pc.max() >= rs.n_instr):
        raise ValueError("sample pc outside the kernel")
    name = rs.kernel_name.encode()
    cats = "\n".join(E.norm_category(c) for c in rs.categories).encode()
    head = _HDR.pack(MAGIC, pc.size, rs.n_instr, rs.period, E.DIALECT_IDX[rs.dialect],
                     len(rs.categories), len(name), len(cats)) + name + cats
    with open(path, "wb") as f:
        f.write(head + b"\0" * (_pad16(len(head)) - len(head)))
        f.write(pc.tobytes())
        f.write(b"\0" * (_pad16(pc.nbytes) - pc.nbytes))
        f.write(cat.tobytes())
        return f.tell()


def read(path, mmap: bool = True) -> RawSamples:
    """Read a sample file; pcs and categories are memory-mapped (no copy)."""
    path = Path(path)
    with open(path, "rb") as f:
        fixed = f.read(_HDR.size)
        magic, n, n_instr, period, d, n_cat, name_len, cat_len = _HDR.unpack(fixed)
        if magic != MAGIC:
            raise ValueError(f"{path}: not a LEO sample file")
        name = f.read(name_len).decode()
        cats = f.read(cat_len).decode()
    off = _pad16(_HDR.size + name_len + cat_len)
    load = (lambda dt, o, c: np.memmap(path, dtype=dt, mode="r", offset=o, shape=(c,))) if mmap and n \
        else (lambda dt, o, c: np.fromfile(path, dtype=dt, count=c, offset=o))
    pc = load(np.int32, off, n)
    cat = load(np.uint8, off + _pad16(4 * n), n)
    return RawSamples(kernel_name=name, dialect=E.DIALECTS[d], period=period, n_instr=n_instr,
                      categories=tuple(cats.split("\n")) if n_cat else (), pc=pc, cat=cat)


def from_profile(ks, pf, counts_by_category=None, seed: int = 0) -> RawSamples:
    """Expand a binned profile (ProfileSoA cls_cnt[N, 8], per CommonStall) into
    a raw stream whose stage-0 binning gives back the same lat / cls_cnt:
    one sample per counted latency sample, categories named by the dialect's
    first vendor category of each CommonStall, order shuffled."""
    cats, first = [], {}
    for name in E.vendor_categories(ks.dialect):
        cs = E.STALL_MAPS[ks.dialect][name]
        if cs not in first:
            first[cs] = len(cats)
            cats.append(name)
    cls = np.asarray(pf.cls_cnt).reshape(-1, 8)
    rows = np.repeat(np.arange(cls.shape[0] * 8), cls.reshape(-1).astype(np.int64))
    pc = (rows // 8).astype(np.int32)
    cs = rows % 8
    cat_of_cs = np.full(8, first.get("other", 0), dtype=np.uint8)
    for name, i in first.items():
        cat_of_cs[E.CS_IDX[name]] = i
    cat = cat_of_cs[cs]
    perm = np.random.default_rng(seed).permutation(pc.size)
    return RawSamples(kernel_name=ks.name, dialect=ks.dialect, period=int(pf.period),
                      n_instr=ks.n_instr, categories=tuple(cats), pc=pc[perm], cat=cat[perm])
