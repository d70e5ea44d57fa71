import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

GOLDEN = ROOT / "tests" / "golden"
GOLDEN_FILES = ("corpus_c1.npz", "reference_suite.npz", "random.npz", "synth.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_cases():
    import golden_io
    out = {}
    for f in GOLDEN_FILES:
        out[f] = golden_io.load(GOLDEN / f)
    return out
