"""The oracle pinned to the REFERENCE at full size (CPU): the C restatement's
outputs on the full C2 / C3 / C5 workloads and on the C4_SUBSET kernels
equal the reference's (tests/golden/full_digests.json, made by running
stalltrace here: tests/golden/make_full.py).  This closes the gap between the
golden sizes (<= a few thousand instructions) and the configs the GPU path
is benchmarked on: the oracle's query-based reaching-definitions formulation
and its sync / DFS walkers are checked against the reference's worklist and
chain walkers on exactly those inputs."""

import json

import pytest

import digest
import parity
from conftest import GOLDEN

FULL = json.loads((GOLDEN / "full_digests.json").read_text())


def oracle_digest(wl):
    from oracle import oracle
    from paper_2604_20032_b200 import synth
    ks = wl.kernel
    o = oracle.run(ks, synth.bin_host(wl))
    return digest.digests(parity.oracle_outputs(ks, o))


@pytest.mark.parametrize("tag", ["c2", "c3", "c5"])
def test_oracle_full_config_matches_reference(tag):
    from paper_2604_20032_b200 import synth
    if tag not in FULL:
        pytest.skip(f"no reference digest for {tag} (tests/golden/make_full.py {tag})")
    errs = digest.compare(FULL[tag], oracle_digest(synth.config_workload(tag)))
    assert not errs, errs


def test_oracle_c4_subset_matches_reference():
    from paper_2604_20032_b200 import synth
    lines = synth.LineTable(4096, seed=999)
    keys = sorted((int(k[3:]) for k in FULL if k.startswith("c4_")))
    assert len(keys) >= 10
    bad = []
    for k in keys:
        errs = digest.compare(FULL[f"c4_{k}"], oracle_digest(synth.c4_kernel(k, lines)))
        if errs:
            bad.append((k, errs[:2]))
    assert not bad, bad
