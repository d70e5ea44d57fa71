"""Pin the C oracle to the reference: every golden vector (produced by running
the reference stalltrace package, tests/golden/make_golden.py) must be
reproduced bit-exactly — edges, pruned edges + valid paths, diagnostics,
slice levels, blame cycles and factors (rel 0), line totals."""

import numpy as np
import pytest

import golden_io
import parity
from conftest import GOLDEN, GOLDEN_FILES
from oracle import oracle


@pytest.mark.parametrize("fname", GOLDEN_FILES)
def test_oracle_matches_reference_golden(fname, golden_cases):
    cases = golden_cases[fname]
    assert cases, fname
    bad = []
    for ks, pf, cfg, exp in cases:
        r = oracle.run(ks, pf, golden_io.config_of(cfg, ks.dialect))
        errs = parity.compare(exp, parity.oracle_outputs(ks, r), rel=0.0, line_rel=1e-12)
        if errs:
            bad.append((ks.name, errs[:2]))
    assert not bad, f"{len(bad)}/{len(cases)} cases differ; first: {bad[:3]}"


def test_oracle_binning_matches_bincount():
    from paper_2604_20032_b200 import synth
    wl = synth.config_workload("c2", scale=0.05)
    lat, cls = oracle.bin_samples(wl.pc, wl.cat, wl.lut, wl.kernel.n_instr)
    ref = synth.bin_host(wl)
    assert np.array_equal(lat, ref.lat)
    assert np.array_equal(cls, ref.cls_cnt)
    assert int(lat.sum()) == wl.n_samples
