"""The reference's OWN test modules, re-pointed at the drop-in:
`pkg/tests/test_depgraph.py`, `test_sync.py`, `test_pruning.py`,
`test_blame.py` and `test_report.py::TestRankHotspots`-style calls run with
every analyzer function they import (build_graph, reaching_definitions,
per_use_link, liveness_filter, trace_*, run_pruning, prune_*,
attribute_blame, self_blame, trace_chain, single_dep_coverage,
rank_hotspots, dump_graph) bound to paper_2604_20032_b200.api, i.e. computed
on the GPU (tests/ref_repoint.py).  They exercise what the golden vectors do
not: stages chained on already-pruned graphs, hand-built DependencyGraphs
(test_blame.py:30-56), self_blame of arbitrary instructions, the dataflow
sub-steps.

Needs the test-only reference install in baseline/_ref
(tools/install_reference.sh; git-ignored, travels to the GPU box)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
SUITE = REF / "stalltrace_tests"

MODULES = ["test_depgraph.py", "test_sync.py", "test_pruning.py", "test_blame.py", "test_report.py"]


@pytest.mark.parametrize("module", MODULES)
def test_reference_suite_on_the_gpu_path(module):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not (SUITE / module).exists():
        pytest.skip("reference not installed in baseline/_ref (run tools/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT), str(ROOT / "tests"), str(SUITE)])
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "ref_repoint", "-p", "no:cacheprovider",
           "--rootdir", str(SUITE), str(SUITE / module)]
    r = subprocess.run(cmd, cwd=str(SUITE), env=env, capture_output=True, text=True, timeout=1800)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert "intact=True" in r.stdout, "the re-pointing plugin did not load (or was undone)"
    assert " passed" in r.stdout, tail
