"""Loader for the in-tree CUDA library libleo_b200.so.

There is no CPU fallback: if the library is missing or cannot be loaded the
import fails loudly (build it with `python -m paper_2604_20032_b200.build` or
`__graft_entry__.build()`).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import abi

LIB_PATH = Path(__file__).resolve().parent / "libleo_b200.so"
# A/B timing of library variants (profiling only): LEO_LIB_VARIANT=<path>
if os.environ.get("LEO_LIB_VARIANT"):
    LIB_PATH = Path(os.environ["LEO_LIB_VARIANT"]).resolve()
ABI_VERSION = 4

_lib = None

# every analysis entry point include/leo_b200.h declares (tests/test_abi.py)
ENTRY_POINTS = ("leo_bin_samples", "leo_build_graph", "leo_prune", "leo_slice", "leo_blame",
                "leo_analyze", "leo_report", "leo_self_blame", "leo_coverage", "leo_rank_hotspots",
                "leo_trace_chain", "leo_liveness_filter", "leo_reaching_definitions",
                "leo_line_rollup", "leo_line_compact")


class LeoLibraryError(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise LeoLibraryError(f"{LIB_PATH} not built; run __graft_entry__.build() "
                              "(no CPU fallback exists for the analysis path)")
    L = C.CDLL(str(LIB_PATH))
    if L.leo_abi_version() != ABI_VERSION:
        raise LeoLibraryError("libleo_b200.so ABI version mismatch; rebuild")
    P = C.c_void_p
    L.leo_bin_samples.argtypes = [C.POINTER(abi.LeoSamples), C.c_int32, P, P, P, P]
    L.leo_build_graph.argtypes = [C.POINTER(abi.LeoKernel), C.POINTER(abi.LeoCaps),
                                  C.POINTER(abi.LeoEdges), C.POINTER(abi.LeoDiags), P, P]
    L.leo_prune.argtypes = [C.POINTER(abi.LeoKernel), C.POINTER(abi.LeoProfile),
                            C.POINTER(abi.LeoConfig), C.POINTER(abi.LeoEdges),
                            C.POINTER(abi.LeoPaths), C.POINTER(abi.LeoEdges),
                            C.POINTER(abi.LeoPaths), C.POINTER(abi.LeoDiags), P, P]
    L.leo_self_blame.argtypes = [C.POINTER(abi.LeoKernel), C.POINTER(abi.LeoProfile),
                                 C.POINTER(abi.LeoEdges), C.c_int32, P, P, P, P]
    L.leo_coverage.argtypes = [C.POINTER(abi.LeoKernel), C.POINTER(abi.LeoEdges), P, P]
    L.leo_rank_hotspots.argtypes = [C.POINTER(abi.LeoKernel), C.POINTER(abi.LeoProfile),
                                    C.c_int32, C.c_int32, P, P, P]
    L.leo_trace_chain.argtypes = [C.POINTER(abi.LeoKernel), C.c_int32, P, P, P, C.c_int32,
                                  C.c_int32, P, P, P, P, P]
    L.leo_line_rollup.argtypes = [C.POINTER(abi.LeoKernel), C.POINTER(abi.LeoProfile), C.c_int32,
                                  P, P, P, P, C.c_int32, P, P, P]
    L.leo_line_compact.argtypes = [P, P, C.c_int32, C.c_int32, P, P, P, P, P]
    L.leo_liveness_filter.argtypes = [C.POINTER(abi.LeoKernel), C.POINTER(abi.LeoEdges), P, P]
    L.leo_reaching_definitions.argtypes = [C.POINTER(abi.LeoKernel), C.POINTER(abi.LeoCaps),
                                           C.POINTER(abi.LeoReachIn), P, P]
    L.leo_slice.argtypes = [C.POINTER(abi.LeoKernel), C.POINTER(abi.LeoProfile),
                            C.POINTER(abi.LeoEdges), P, P, P]
    L.leo_blame.argtypes = [C.POINTER(abi.LeoKernel), C.POINTER(abi.LeoProfile),
                            C.POINTER(abi.LeoEdges), C.POINTER(abi.LeoPaths),
                            C.POINTER(abi.LeoEdges), P, C.c_int32, C.POINTER(abi.LeoBlame),
                            P, P, P, P]
    L.leo_analyze.argtypes = [C.POINTER(abi.LeoKernel), C.POINTER(abi.LeoProfile),
                              C.POINTER(abi.LeoSamples), C.POINTER(abi.LeoConfig),
                              C.POINTER(abi.LeoCaps), C.POINTER(abi.LeoEdges),
                              C.POINTER(abi.LeoEdges), C.POINTER(abi.LeoPaths),
                              C.POINTER(abi.LeoDiags), C.POINTER(abi.LeoBlame), P, P, P,
                              C.c_int32, P, P, P, P]
    L.leo_report.argtypes = [C.POINTER(abi.LeoKernel), C.POINTER(abi.LeoProfile),
                             C.POINTER(abi.LeoEdges), C.POINTER(abi.LeoEdges),
                             C.POINTER(abi.LeoBlame), C.POINTER(abi.LeoReport), P, P]
    L.leo_kernel_name.argtypes = [C.c_int]
    L.leo_debug_phases.argtypes = [C.c_int32, P, C.c_int32]
    L.leo_debug_phases.restype = C.c_int
    L.leo_kernel_name.restype = C.c_char_p
    L.leo_events_create.argtypes = [C.c_int32, P]
    L.leo_events_elapsed.argtypes = [C.c_int32, P, P, P]
    L.leo_events_destroy.argtypes = [C.c_int32, P]
    for f in ("leo_events_create", "leo_events_elapsed", "leo_events_destroy"):
        getattr(L, f).restype = C.c_int
    for f in ENTRY_POINTS:
        getattr(L, f).restype = C.c_int
    _lib = L
    return L


def check(rc: int, what: str):
    if rc != 0:
        if rc <= -1000:
            raise LeoLibraryError(f"{what}: CUDA error {-(rc + 1000)}")
        raise ValueError(f"{what}: invalid arguments (code {rc})")
