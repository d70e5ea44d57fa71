"""GPU parity: the CUDA path (libleo_b200.so through its C ABI) against the
reference's golden vectors and the oracle.

Bit-exact: base edges, pruned edges, valid paths, diagnostics, slice levels,
blame structure, blame cycles and factors (the device reproduces the
reference's floating-point evaluation order; north-star tolerance is 1e-6
relative, we test rel=0).  Per-line totals use FP64 atomics on the device
(summation order differs): rel 1e-9.
"""

import numpy as np
import pytest

import golden_io
import parity
from conftest import GOLDEN_FILES

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def device_outputs(ks, r):
    from paper_2604_20032_b200 import diagnostics
    got = dict(bprod=r["bprod"], bcons=r["bcons"], bmeta=r["bmeta"], pprod=r["pprod"],
               pcons=r["pcons"], pmeta=r["pmeta"], npaths=r["npaths"], first=r["first"],
               plen=r["plen"], pacc=r["pacc"], level=r["level"],
               line_blame=r["line_blame"], line_stall=r["line_stall"])
    got["diags"] = list(ks.prefix_diagnostics) + diagnostics.render(ks.dialect, ks.offset,
                                                                    r["diag_records"])
    got.update(parity.blame_arrays(ks.dialect, r["e_stalled"], r["e_edge"], r["e_sub"],
                                   r["e_blame"], r["e_factors"], r["pprod"], r["pmeta"]))
    return got


@pytest.fixture(scope="module")
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_20032_b200 import _lib
    _lib.lib()          # fail loudly if the library is missing
    return torch.device("cuda:0")


@pytest.mark.parametrize("fname", GOLDEN_FILES)
def test_device_matches_reference_golden(fname, golden_cases, cuda):
    from paper_2604_20032_b200 import device
    cases = golden_cases[fname]
    bad = []
    for ks, pf, cfg, exp in cases:
        r = device.analyze_soa(ks, pf, golden_io.config_of(cfg, ks.dialect), device=cuda)
        assert r["status"] == 0, (ks.name, r["status"])
        errs = parity.compare(exp, device_outputs(ks, r), rel=0.0, line_rel=1e-9)
        if errs:
            bad.append((ks.name, errs[:2]))
    assert not bad, f"{len(bad)}/{len(cases)} cases differ; first: {bad[:3]}"


@pytest.mark.parametrize("tag,scale", [("c2", 1.0), ("c3", 1.0), ("c5", 0.05)])
def test_device_matches_oracle_synthetic(tag, scale, cuda):
    """Full-size C2/C3 (C5 at 5 %): raw samples binned on the device, whole
    pipeline, compared with the oracle on the same seeded inputs."""
    from oracle import oracle
    from paper_2604_20032_b200 import abi, device, synth
    wl = synth.config_workload(tag, scale=scale)
    ks = wl.kernel
    r = device.analyze_soa(ks, wl.profile, abi.make_config(dialect=ks.dialect),
                           samples=(wl.pc, wl.cat, wl.lut), device=cuda)
    assert r["status"] == 0
    pf = synth.bin_host(wl)
    assert np.array_equal(r["lat"], pf.lat)
    assert np.array_equal(r["cls_cnt"], pf.cls_cnt)
    o = oracle.run(ks, pf)
    exp = parity.oracle_outputs(ks, o)
    errs = parity.compare(exp, device_outputs(ks, r), rel=0.0, line_rel=1e-9)
    assert not errs, errs
    # conservation (report.py:147-155): per-line blame sums to total stall cycles
    total = float((pf.lat.astype(np.int64) * pf.period).sum())
    assert np.isclose(r["line_blame"].sum(), total, rtol=1e-9)
    assert np.isclose(r["line_stall"].sum(), total, rtol=1e-9)


@pytest.mark.parametrize("tag,knobs", [
    ("c2", {"LEO_SYNC_FORK_AT": "0", "LEO_RU_PARTS": "3", "LEO_WC_CTAS": "148", "LEO_PRUNE_THREADS": "128"}),
    ("c2", {"LEO_WC_STEPS": "32", "LEO_NO_PRIO": "1"}),
    ("c2", {"LEO_WC_STEPS": "16", "LEO_WC_CTA": "1"}),
    ("c3", {"LEO_SYNC_FORK_AT": "2", "LEO_RU_PARTS": "1", "LEO_PRUNE_THREADS": "128"}),
    ("c3", {"LEO_SETTER_GLOBAL": "1"}),
    ("c5", {"LEO_SETTER_GLOBAL": "1"}),
    ("c5", {"LEO_T1": "0", "LEO_BIN_SLOTS": "8192", "LEO_BIN_PROBE": "8"}),
    ("c5", {"LEO_T1": "1", "LEO_BIN_SLOTS": "26624", "LEO_BIN_PROBE": "4", "LEO_SCAN_TILED": "1"}),
    ("c5", {"LEO_T1": "3", "LEO_BLAME_2PASS": "1", "LEO_BIN_LOWPRIO": "1", "LEO_MP_COOP": "1"}),
    ("c2", {"LEO_BLAME_2PASS": "1", "LEO_SCAN_TILED": "1", "LEO_WC_CLUSTER": "1", "LEO_MP_COOP": "1"}),
    ("c2", {"LEO_WC_CLUSTER": "8", "LEO_WC_CTAS": "64", "LEO_BLAME_SPLIT": "1"}),
    ("c5", {"LEO_BLAME_UNSPLIT": "1", "LEO_BIN_SLOTS": "8192", "LEO_BIN_PROBE": "4"}),
    ("c3", {"LEO_BLAME_SPLIT": "1"}),
])
def test_device_schedule_knobs_exact(tag, knobs, cuda, monkeypatch):
    """The scheduling knobs (fork points, CTAs per unit, waitcnt tier size
    and step limit, prune CTA size, tier-1 reach table geometry, binning
    table geometry, one- vs two-pass blame, one-launch vs tiled scans) move
    work between tiers and branches; the results must not move.  Half-size
    C2 / C3 and 5 % C5 against the oracle."""
    from oracle import oracle
    from paper_2604_20032_b200 import abi, device, synth
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    wl = synth.config_workload(tag, scale=0.05 if tag == "c5" else 0.5)
    ks = wl.kernel
    r = device.analyze_soa(ks, wl.profile, abi.make_config(dialect=ks.dialect),
                           samples=(wl.pc, wl.cat, wl.lut), device=cuda)
    assert r["status"] == 0
    pf = synth.bin_host(wl)
    o = oracle.run(ks, pf)
    errs = parity.compare(parity.oracle_outputs(ks, o), device_outputs(ks, r), rel=0.0, line_rel=1e-9)
    assert not errs, errs


def test_device_full_c5_properties(cuda):
    """C5 at full size (1M instructions, 100M samples): size-independent
    properties — binning conserves S, blame conserves stall cycles per line
    and in total, every stalled PC is in the slice at level 0, slice levels
    are consistent with pruned edges (each level-L node has a consumer at L-1)."""
    from paper_2604_20032_b200 import abi, device, synth
    wl = synth.config_workload("c5")
    ks = wl.kernel
    r = device.analyze_soa(ks, wl.profile, abi.make_config(dialect="nvidia"),
                           samples=(wl.pc, wl.cat, wl.lut), device=cuda)
    assert r["status"] == 0
    lat = r["lat"].astype(np.int64)
    assert lat.sum() == wl.n_samples
    total = float((lat * 100).sum())
    assert np.isclose(r["e_blame"].sum(), total, rtol=1e-9)
    assert np.isclose(r["line_blame"].sum(), total, rtol=1e-9)
    lv = r["level"]
    assert np.all(lv[lat > 0] == 0) and np.all(lv[lat == 0] != 0)
    pp, pc = r["pprod"], r["pcons"]
    deeper = lv[pp] > 0
    # every producer at level L>0 was reached from a consumer at level L-1
    best = np.full(ks.n_instr, np.iinfo(np.int32).max, dtype=np.int64)
    ok = (lv[pc] >= 0)
    np.minimum.at(best, pp[ok], lv[pc[ok]].astype(np.int64) + 1)
    inside = lv >= 0
    assert np.all(best[inside & (lv > 0)] == lv[inside & (lv > 0)])
    assert deeper.sum() >= 0


@pytest.mark.parametrize("flags", [1, 2 | 4 | 8 | 16, 32])
@pytest.mark.parametrize("fname", ["corpus_c1.npz", "random.npz", "synth.npz"])
def test_device_fallback_tiers_match_golden(fname, flags, golden_cases, cuda):
    """Every work item forced onto the larger tiers (warp / global-scratch
    reach search, exact sync walker, global-scratch DFS, global self-blame BFS)
    must give the same bits as the fast tiers."""
    from paper_2604_20032_b200 import device
    bad = []
    for ks, pf, cfg, exp in golden_cases[fname]:
        r = device.analyze_soa(ks, pf, golden_io.config_of(cfg, ks.dialect), device=cuda,
                               debug_flags=flags)
        errs = parity.compare(exp, device_outputs(ks, r), rel=0.0, line_rel=1e-9)
        if errs:
            bad.append((ks.name, errs[:2]))
    assert not bad, f"{len(bad)} cases differ with debug flags {flags}; first: {bad[:3]}"


@pytest.mark.parametrize("tag,scale,world", [("c5", 0.05, 3), ("c2", 1.0, 2)])
def test_device_consumer_shards_recombine(tag, scale, world, cuda):
    """Stalled-PC sharding on the device (LeoConfig.consumer_lo/hi + samples
    partitioned by owner of pc): per-rank blame entries concatenated in rank
    order equal the unsharded entries bit-exactly; summed per-line vectors
    equal the unsharded totals; per-rank pruned edges are exactly the
    unsharded pruned edges whose consumer the rank owns."""
    from paper_2604_20032_b200 import abi, device, synth
    from paper_2604_20032_b200 import dist as D
    wl = synth.config_workload(tag, scale=scale)
    ks = wl.kernel
    full = device.analyze_soa(ks, wl.profile, abi.make_config(dialect=ks.dialect),
                              samples=(wl.pc, wl.cat, wl.lut), device=cuda)
    ranges = D.consumer_ranges(ks, world)
    parts = D.partition_samples(wl.pc, ranges)
    st, bl, sub, cause, lb, ls = [], [], [], [], 0.0, 0.0
    for (lo, hi), idx in zip(ranges, parts):
        r = device.analyze_soa(ks, wl.profile,
                               abi.make_config(dialect=ks.dialect, consumer_range=(lo, hi)),
                               samples=(wl.pc[idx], wl.cat[idx], wl.lut), device=cuda)
        assert r["status"] == 0
        st.append(r["e_stalled"])
        bl.append(r["e_blame"])
        sub.append(r["e_sub"])
        cause.append(r["e_cause"])
        lb = lb + r["line_blame"]
        ls = ls + r["line_stall"]
        own = (full["pcons"] >= lo) & (full["pcons"] < hi)
        got = set(zip(r["pprod"].tolist(), r["pcons"].tolist(), r["pmeta"].tolist()))
        exp = set(zip(full["pprod"][own].tolist(), full["pcons"][own].tolist(),
                      full["pmeta"][own].tolist()))
        assert got == exp
    assert np.array_equal(np.concatenate(st), full["e_stalled"])
    assert np.array_equal(np.concatenate(bl), full["e_blame"])
    # self-blame subcategories too: the indirect-addressing test of an owned
    # instruction walks RAW edges of instructions other ranks own
    assert np.array_equal(np.concatenate(sub), full["e_sub"])
    assert np.array_equal(np.concatenate(cause), full["e_cause"])
    assert np.allclose(lb, full["line_blame"], rtol=1e-9, atol=1e-6)
    assert np.allclose(ls, full["line_stall"], rtol=1e-9, atol=1e-6)


def test_device_batch_matches_per_kernel_oracle(cuda):
    """C4-style batch (kernels concatenated per dialect, one pipeline pass on
    the device): every kernel's slice of the batch result equals the oracle
    on that kernel alone."""
    from oracle import oracle
    from paper_2604_20032_b200 import abi, device, synth
    from paper_2604_20032_b200 import batch as BT
    lines = synth.LineTable(256, seed=999)
    for dialect in ("nvidia", "amd", "intel"):
        wls = [synth.make_workload(dialect, 2000, 10_000, 7000 + s, lines=lines, name=f"k{s}")
               for s in range(12)]
        b = BT.concat(wls)
        r = device.analyze_soa(b.kernel, b.profile, abi.make_config(dialect=dialect),
                               samples=(b.pc, b.cat, b.lut), device=cuda)
        assert r["status"] == 0
        for wl, got in zip(wls, BT.split_result(b, r)):
            o = oracle.run(wl.kernel, synth.bin_host(wl))
            for f, e in (("bprod", o.prod), ("bmeta", o.meta), ("pprod", o.p_prod),
                         ("pmeta", o.p_meta), ("e_stalled", o.e_stalled), ("e_blame", o.e_blame),
                         ("level", o.level)):
                assert np.array_equal(got[f], e), (dialect, wl.kernel.name, f)

@pytest.mark.parametrize("width", [4, 3])
@pytest.mark.parametrize("tag,scale", [("c2", 0.2), ("c5", 0.05), ("c3", 1.0)])
def test_packed_and_split_sample_streams_agree(tag, scale, width, cuda):
    """The packed stream (one u32 word per sample, or the 3-byte words of
    packed_bytes = 3) bins to the same counts and the same analysis as the
    pc / cat arrays, on the small-stream kernel (C2 scale) and the one-pass
    hash (5 M samples); the stream is cut to a length that is not a multiple
    of 4 so the tail path runs too."""
    from paper_2604_20032_b200 import abi, device, synth
    wl = synth.config_workload(tag, scale=scale)
    cfg = abi.make_config(dialect=wl.kernel.dialect)
    n = len(wl.pc) - 3
    smp = (wl.pc[:n], wl.cat[:n], wl.lut)
    a = device.analyze_soa(wl.kernel, wl.profile, cfg, samples=smp, device=cuda, packed=True, width=width)
    b = device.analyze_soa(wl.kernel, wl.profile, cfg, samples=smp, device=cuda, packed=False)
    assert a["status"] == 0 and b["status"] == 0
    for key in ("lat", "cls_cnt", "bprod", "bmeta", "pprod", "e_stalled", "e_blame", "level"):
        assert np.array_equal(a[key], b[key]), key
