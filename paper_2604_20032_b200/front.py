"""Native listing front-end: listing text -> KernelSoA.

Drop-in for the reference's host front-end of the hot path's inputs,
`disasm.parse_kernels` (disasm.py:618-626, parse_listing :259-409, build_cfg
:495-607) followed by `soa.encode_cfg`: libleo_front.so (C++,
native/leo_front.cpp) parses the text and emits the structure-of-arrays the
device library consumes, so no per-instruction Python objects are built.
Errors raise `ListingError` with the reference's message text.

The opcode classification table is an input (isa.py OpcodeTable format), as
the reference's `table` argument is; `default_table_text(dialect)` returns
the reference's bundled table when `stalltrace` is importable.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from . import enums as E
from .soa import KernelSoA

LIB_PATH = Path(__file__).resolve().parent / "libleo_front.so"
_L = None


class ListingError(ValueError):
    """disasm ListingError (errors.py:15-30): message carries token / line / column."""


def lib():
    global _L
    if _L is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} missing: run paper_2604_20032_b200.build")
        L = C.CDLL(str(LIB_PATH))
        P = C.c_void_p
        L.leo_front_parse.restype = P
        L.leo_front_parse.argtypes = [C.c_int32, C.c_char_p, C.c_int64, C.c_char_p, C.c_int64]
        L.leo_front_error.argtypes = [P, C.c_char_p, C.c_int32]
        L.leo_front_error.restype = C.c_int32
        L.leo_front_n_kernels.argtypes = [P]
        L.leo_front_kernel_name.argtypes = [P, C.c_int32]
        L.leo_front_kernel_name.restype = C.c_char_p
        L.leo_front_sizes.argtypes = [P, C.c_int32, P]
        L.leo_front_arrays.argtypes = [P, C.c_int32] + [P] * 16
        L.leo_front_string.argtypes = [P, C.c_int32, C.c_int32, C.c_int32]
        L.leo_front_string.restype = C.c_char_p
        L.leo_front_strings.argtypes = [P, C.c_int32, C.c_int32, C.c_char_p, C.c_int64]
        L.leo_front_strings.restype = C.c_int64
        L.leo_front_free.argtypes = [P]
        _L = L
    return _L


def default_table_text(dialect: str) -> str:
    """The reference's bundled opcode table (needs `stalltrace`)."""
    from importlib import resources
    return resources.files("stalltrace").joinpath(f"data/{dialect}.opcodes").read_text(encoding="utf-8")


def parse_kernels_soa(dialect: str, text: str, table_text: str | None = None) -> dict:
    """{kernel name: (KernelSoA, meta)} with meta = mnemonics, src_locs
    (str(SourceLoc) or None) and the CFG diagnostics, in section order."""
    L = lib()
    if table_text is None:
        table_text = default_table_text(dialect)
    t = text.encode()
    tb = table_text.encode()
    h = L.leo_front_parse(E.DIALECT_IDX[dialect], t, len(t), tb, len(tb))
    try:
        n = L.leo_front_error(h, None, 0)
        if n:
            buf = C.create_string_buffer(n + 1)
            L.leo_front_error(h, buf, n + 1)
            raise ListingError(buf.value.decode())
        out = {}
        for k in range(L.leo_front_n_kernels(h)):
            sz = np.zeros(8, dtype=np.int64)
            L.leo_front_sizes(h, k, sz.ctypes.data)
            N, B, M, ES, EP, U, NL, ND = (int(x) for x in sz)
            a = dict(opclass=np.zeros(N, np.uint8), block_of=np.zeros(N, np.int32),
                     opnd_ptr=np.zeros(N + 1, np.int32), opnd=np.zeros(M, np.uint32),
                     sync_kind=np.zeros(N, np.uint8), sync_a=np.zeros(N, np.uint32),
                     sync_b=np.zeros(N, np.uint32), blk_first=np.zeros(B, np.int32),
                     blk_last=np.zeros(B, np.int32), succ_ptr=np.zeros(B + 1, np.int32),
                     succ=np.zeros(ES, np.int32), pred_ptr=np.zeros(B + 1, np.int32),
                     pred=np.zeros(EP, np.int32), unit_base=np.zeros(8, np.int32),
                     offset=np.zeros(N, np.int64), line_id=np.zeros(N, np.int32))
            L.leo_front_arrays(h, k, *(v.ctypes.data for v in a.values()))
            def strings(which, count):
                if count == 0:
                    return []
                size = L.leo_front_strings(h, k, which, None, 0)
                buf = C.create_string_buffer(max(size, 1))
                L.leo_front_strings(h, k, which, buf, size)
                return buf.raw[:size].decode().split("\n")

            lines = strings(2, NL)
            diags = tuple(strings(3, ND))
            locs = strings(1, N)
            name = L.leo_front_kernel_name(h, k).decode()
            ks = KernelSoA(name=name, dialect=dialect, n_units=U, lines=lines, prefix_diagnostics=diags,
                           **a)
            meta = dict(mnemonics=strings(0, N), src_locs=[x if x else None for x in locs],
                        diagnostics=diags)
            out[name] = (ks, meta)
        return out
    finally:
        L.leo_front_free(h)


# ---------------------------------------------------------------------------
# Profile documents (native/leo_profile.cpp): JSON text -> ProfileSoA.

class ProfileError(ValueError):
    """profile ProfileError (errors.py:33-34): schema / invariant violation."""


class InputError(ValueError):
    """errors.InputError raised by isa.Dialect.from_name for an unknown vendor."""


_PROFILE_FNS = False


def _profile_lib():
    global _PROFILE_FNS
    L = lib()
    if not _PROFILE_FNS:
        P = C.c_void_p
        L.leo_profile_parse.restype = P
        L.leo_profile_parse.argtypes = [C.c_char_p, C.c_int64]
        L.leo_profile_error.restype = C.c_int32
        L.leo_profile_error.argtypes = [P, C.c_char_p, C.c_int32, P]
        L.leo_profile_n_kernels.argtypes = [P]
        L.leo_profile_kernel_name.restype = C.c_char_p
        L.leo_profile_kernel_name.argtypes = [P, C.c_int32]
        L.leo_profile_info.argtypes = [P, C.c_int32, P]
        L.leo_profile_records.argtypes = [P, C.c_int32] + [P] * 6
        L.leo_profile_attach.restype = C.c_int32
        L.leo_profile_attach.argtypes = [P, C.c_int32, C.c_char_p, C.c_int32, C.c_int32] + [P] * 7
        L.leo_profile_diagnostic.restype = C.c_char_p
        L.leo_profile_diagnostic.argtypes = [P]
        L.leo_profile_free.argtypes = [P]
        _PROFILE_FNS = True
    return L


def _raise_profile(L, h):
    n = C.c_int32(0)
    kind = L.leo_profile_error(h, None, 0, C.byref(n))
    if not kind:
        return
    buf = C.create_string_buffer(n.value + 1)
    L.leo_profile_error(h, buf, n.value + 1, None)
    msg = buf.value.decode()
    raise (InputError if kind == 2 else ProfileError)(msg)


class ProfileDoc:
    """A parsed profile document (profile.load_profiles, profile.py:244-263):
    the kernels in document order, each `name`, `dialect`, `period` and its
    records as arrays (`records(k)`), joined to a KernelSoA by `attach`."""

    def __init__(self, text: str):
        self._L = _profile_lib()
        t = text.encode("utf-8", "surrogatepass")
        self._h = self._L.leo_profile_parse(t, len(t))
        try:
            _raise_profile(self._L, self._h)
        except Exception:
            self.close()
            raise
        self.kernels = []
        info = np.zeros(3, dtype=np.int64)
        for k in range(self._L.leo_profile_n_kernels(self._h)):
            self._L.leo_profile_info(self._h, k, info.ctypes.data)
            self.kernels.append((self._L.leo_profile_kernel_name(self._h, k).decode(),
                                 E.DIALECTS[int(info[0])], int(info[1]), int(info[2])))

    def close(self):
        if getattr(self, "_h", None):
            self._L.leo_profile_free(self._h)
            self._h = None

    __del__ = close

    def index(self, name: str) -> int:
        for k, kp in enumerate(self.kernels):
            if kp[0] == name:
                return k
        raise KeyError(name)

    def records(self, k: int) -> dict:
        """Kernel k's records in document order: offset, latency, total and
        exec (-1 = None), efficiency, and counts per common stall class [n, 8]
        (the vendor categories already mapped, profile.py:106-111)."""
        n = self.kernels[k][3]
        r = dict(offset=np.zeros(n, np.int64), lat=np.zeros(n, np.int64),
                 total=np.zeros(n, np.int64), exec_cnt=np.zeros(n, np.int64),
                 eff=np.zeros(n, np.float64), cls_cnt=np.zeros((n, 8), np.int64))
        self._L.leo_profile_records(self._h, k, *(v.ctypes.data for v in r.values()))
        return r

    def attach(self, ks: KernelSoA, k: int | None = None):
        """profile.attach (profile.py:332-366) + soa.encode_profile for one
        kernel: (ProfileSoA, diagnostics tuple).  `k` defaults to the kernel
        named like `ks`; a name or vendor mismatch raises ProfileError."""
        from .soa import ProfileSoA
        if k is None:
            k = self.index(ks.name)
        n = ks.n_instr
        a = dict(lat=np.zeros(n, np.int32), cls_cnt=np.zeros((n, 8), np.int32),
                 exec_cnt=np.zeros(n, np.int64), total=np.zeros(n, np.int32),
                 eff=np.zeros(n, np.float64), sampled=np.zeros(n, np.uint8))
        off = np.ascontiguousarray(ks.offset, dtype=np.int64)
        rc = self._L.leo_profile_attach(self._h, k, ks.name.encode(), E.DIALECT_IDX[ks.dialect], n,
                                        off.ctypes.data, *(v.ctypes.data for v in a.values()))
        if rc:
            _raise_profile(self._L, self._h)
        d = self._L.leo_profile_diagnostic(self._h).decode()
        return ProfileSoA(period=self.kernels[k][2], **a), ((d,) if d else ())


def load_profiles(text: str) -> ProfileDoc:
    """Native profile.load_profiles: parse every kernel object of a document."""
    return ProfileDoc(text)


def load_inputs(dialect: str, listing: str, profile_text: str, table_text: str | None = None,
                kernel: str | None = None, profile_name: str = "<profile>") -> list:
    """The CLI's input stage natively (cli._load_inputs, cli.py:75-111):
    parse_kernels + load_profiles, then attach (profile.py:332-366) for the
    selected kernel or every kernel in name order.  Returns [(KernelSoA,
    ProfileSoA)], each kernel's attach diagnostics prepended to its CFG
    diagnostics as build_graph orders them (depgraph.py:527).  A kernel
    without a profile entry raises InputError, as the CLI does."""
    kernels = parse_kernels_soa(dialect, listing, table_text)
    doc = ProfileDoc(profile_text)
    if kernel is not None:
        if kernel not in kernels:
            raise InputError(f"kernel {kernel!r} not found in the listing")
        names = [kernel]
    else:
        names = sorted(kernels)
    out = []
    for name in names:
        try:
            k = doc.index(name)
        except KeyError:
            raise InputError(f"profile {profile_name} has no entry for kernel {name!r}") from None
        ks = kernels[name][0]
        prof, diags = doc.attach(ks, k)
        ks.prefix_diagnostics = tuple(diags) + tuple(ks.prefix_diagnostics)
        out.append((ks, prof))
    return out
