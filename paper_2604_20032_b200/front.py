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
