"""pytest plugin (-p ref_repoint): re-point the reference's analyzer API at
the CUDA drop-in before the reference's own test modules import it.

Every hot-path name the reference exports (stalltrace/__init__.py:9-64) is
replaced, in `stalltrace` and in the module that defines it, by the
same-named function of paper_2604_20032_b200.api, so
`from stalltrace.analysis import attribute_blame` in a reference test binds
the GPU implementation.  Used by tests/test_ref_suite.py only."""

import stalltrace
import stalltrace.analysis as _an
import stalltrace.depgraph as _dg
import stalltrace.report as _rp

from paper_2604_20032_b200 import api

REPOINTED = {
    _dg: ("build_graph", "reaching_definitions", "per_use_link", "liveness_filter", "trace_waitcnt",
          "trace_barriers", "trace_swsb", "dump_graph"),
    _an: ("run_pruning", "prune_opcode", "prune_barrier", "prune_latency", "prune_execution",
          "attribute_blame", "self_blame", "trace_chain", "single_dep_coverage"),
    _rp: ("rank_hotspots",),
}
for _mod, _names in REPOINTED.items():
    for _n in _names:
        setattr(_mod, _n, getattr(api, _n))
        if hasattr(stalltrace, _n):
            setattr(stalltrace, _n, getattr(api, _n))


def pytest_terminal_summary(terminalreporter):
    n = sum(len(v) for v in REPOINTED.values())
    ok = all(getattr(m, f) is getattr(api, f) for m, fs in REPOINTED.items() for f in fs)
    terminalreporter.write_line(f"ref_repoint: {n} stalltrace functions re-pointed at "
                                f"paper_2604_20032_b200.api (GPU), intact={ok}")
