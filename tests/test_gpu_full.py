"""Full-size parity on every BASELINE config (north star: "bit-exact slices
and pruned graphs versus the CPU oracle on all five configs").

  * C2 (10k AMD, 1M samples), C3 (50k Intel, 5M samples) and C5 (1M NVIDIA,
    100M samples) at FULL size: raw samples binned on the device, the whole
    pipeline, compared with the REFERENCE's own outputs on the same seeded
    inputs through per-field digests (tests/golden/full_digests.json, made by
    tests/golden/make_full.py running stalltrace here) and with the oracle
    field by field (diagnosable diffs).
  * C4: the whole 2,000 x 20,000-instruction batch (kernels concatenated per
    dialect, one device pass per dialect), every kernel's slice of the result
    against the oracle on that kernel alone, and the reference digests of the
    C4_SUBSET kernels.
  * C5 slice properties the digests also imply, stated directly: closure
    (every producer of a pruned edge into the slice is in the slice) and
    minimality of levels.
"""

import json
import os
from concurrent.futures import ProcessPoolExecutor, ThreadPoolExecutor

import numpy as np
import pytest

import digest
import parity
from conftest import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FULL = json.loads((GOLDEN / "full_digests.json").read_text())


@pytest.fixture(scope="module")
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_20032_b200 import _lib
    _lib.lib()
    return torch.device("cuda:0")


def device_fields(ks, r):
    from test_gpu_parity import device_outputs
    return device_outputs(ks, r)


def run_full(tag, cuda):
    from paper_2604_20032_b200 import abi, device, synth
    wl = synth.config_workload(tag)
    ks = wl.kernel
    r = device.analyze_soa(ks, wl.profile, abi.make_config(dialect=ks.dialect),
                           samples=(wl.pc, wl.cat, wl.lut), device=cuda)
    assert r["status"] == 0
    return wl, r


@pytest.mark.parametrize("tag", ["c2", "c3", "c5"])
def test_full_size_matches_reference_and_oracle(tag, cuda):
    from oracle import oracle
    from paper_2604_20032_b200 import synth
    wl, r = run_full(tag, cuda)
    ks = wl.kernel
    pf = synth.bin_host(wl)
    assert np.array_equal(r["lat"], pf.lat) and np.array_equal(r["cls_cnt"], pf.cls_cnt)
    got = device_fields(ks, r)
    # 1. the oracle, field by field (diagnosable)
    o = oracle.run(ks, pf)
    errs = parity.compare(parity.oracle_outputs(ks, o), got, rel=0.0, line_rel=1e-9)
    # 2. the reference's own outputs on the same inputs (digests)
    errs += digest.compare(FULL[tag], digest.digests(got))
    assert not errs, errs
    meta = FULL[tag]["_meta"]
    assert (len(r["bprod"]), len(r["pprod"]), len(r["e_stalled"])) == \
        (meta["edges"], meta["pruned"], meta["entries"])


def test_full_c5_slice_closure(cuda):
    """Slice = backward closure from every stalled PC over the pruned edges:
    (i) stalled PCs are at level 0 and nothing else is; (ii) closure: the
    producer of every pruned edge whose consumer is in the slice is in the
    slice; (iii) minimality: a member at level L > 0 has a pruned out-edge to
    a member at level L - 1 and none to a member below L - 1."""
    wl, r = run_full("c5", cuda)
    lat = r["lat"].astype(np.int64)
    assert lat.sum() == wl.n_samples
    total = float((lat * 100).sum())
    assert np.isclose(r["e_blame"].sum(), total, rtol=1e-9)
    assert np.isclose(r["line_blame"].sum(), total, rtol=1e-9)
    lv = r["level"].astype(np.int64)
    assert np.all(lv[lat > 0] == 0) and np.all(lv[lat == 0] != 0)
    pp, pc = r["pprod"], r["pcons"]
    into = lv[pc] >= 0
    assert np.all(lv[pp[into]] >= 0), "a producer of an in-slice consumer is missing from the slice"
    best = np.full(wl.kernel.n_instr, np.iinfo(np.int64).max, dtype=np.int64)
    np.minimum.at(best, pp[into], lv[pc[into]] + 1)
    deep = lv > 0
    assert np.all(best[deep] == lv[deep])
    assert np.all(lv[(lv >= 0) & (best < np.iinfo(np.int64).max)]
                  <= best[(lv >= 0) & (best < np.iinfo(np.int64).max)])


def _c4_kernel(k):
    from paper_2604_20032_b200 import synth
    return synth.c4_kernel(k, synth.LineTable(4096, seed=999))


def test_full_c4_batch_matches_oracle_and_reference(cuda):
    """The whole C4 batch: 2,000 kernels x 20,000 instructions, 100k samples
    each (200 M samples), three dialect batches on one GPU."""
    from oracle import oracle
    from paper_2604_20032_b200 import abi, device, synth
    from paper_2604_20032_b200 import batch as BT
    K = synth.C4_KERNELS
    with ProcessPoolExecutor(min(16, os.cpu_count() or 1)) as ex:
        wls = list(ex.map(_c4_kernel, range(K), chunksize=25))
    groups = {}
    for k, wl in enumerate(wls):
        groups.setdefault(BT.group_key(wl), []).append(k)
    per_kernel = {}
    line_blame = None
    for key in sorted(groups):
        ids = groups[key]
        b = BT.concat([wls[k] for k in ids])
        r = device.analyze_soa(b.kernel, b.profile, abi.make_config(dialect=key[0]),
                               samples=(b.pc, b.cat, b.lut), device=cuda)
        assert r["status"] == 0, (key, r["status"])
        line_blame = r["line_blame"] if line_blame is None else line_blame + r["line_blame"]
        for k, d in zip(ids, BT.split_result(b, r)):
            per_kernel[k] = d
        del r, b
    assert len(per_kernel) == K

    def check(k):
        wl = wls[k]
        ks = wl.kernel
        pf = synth.bin_host(wl)
        o = oracle.run(ks, pf)
        d = per_kernel[k]
        d["line_blame"], d["line_stall"] = o.line_blame, o.line_stall   # batch-wide vectors, checked below
        got = device_fields(ks, d)
        errs = parity.compare(parity.oracle_outputs(ks, o), got, rel=0.0, line_rel=1e-9,
                              parts=("base", "pruned", "diags", "blame", "slice"))
        ref = FULL.get(f"c4_{k}")
        if ref is not None:
            dg = digest.digests(got)
            errs += [e for e in digest.compare(ref, dg) if not e.startswith("line_")]
        return k, errs, o.line_blame

    bad, lb_sum = [], 0.0
    with ThreadPoolExecutor(min(16, os.cpu_count() or 1)) as ex:      # the C oracle drops the GIL
        for k, errs, lb in ex.map(check, range(K)):
            if errs:
                bad.append((k, errs[:2]))
            lb_sum = lb_sum + lb
    assert not bad, f"{len(bad)}/{K} C4 kernels differ; first: {bad[:3]}"
    assert np.allclose(line_blame, lb_sum, rtol=1e-9, atol=1e-6)
    assert sum(1 for k in range(K) if f"c4_{k}" in FULL) >= 10
