"""Binary raw-sample format: round trip, category
mapping, profile expansion (CPU); file -> pinned -> device binning (GPU)."""

import numpy as np
import pytest

import golden_io


def _c2(scale=0.05):
    from paper_2604_20032_b200 import synth
    return synth.config_workload("c2", scale=scale)


def test_roundtrip_and_lut(tmp_path):
    from paper_2604_20032_b200 import enums as E
    from paper_2604_20032_b200 import samples
    wl = _c2()
    rs = samples.RawSamples(kernel_name="k", dialect="amd", period=wl.profile.period,
                            n_instr=wl.kernel.n_instr, categories=E.vendor_categories("amd"),
                            pc=wl.pc, cat=wl.cat)
    p = tmp_path / "s.leosmp"
    size = samples.write(p, rs)
    assert size >= wl.pc.nbytes + wl.cat.nbytes
    back = samples.read(p)
    assert back.kernel_name == "k" and back.dialect == "amd" and back.n_instr == wl.kernel.n_instr
    assert np.array_equal(back.pc, wl.pc) and np.array_equal(back.cat, wl.cat)
    assert np.array_equal(back.lut(), wl.lut)
    empty = samples.RawSamples("e", "nvidia", 10, 3, (), np.zeros(0, np.int32), np.zeros(0, np.uint8))
    samples.write(tmp_path / "e.leosmp", empty)
    assert samples.read(tmp_path / "e.leosmp").n_samples == 0
    with pytest.raises(ValueError):
        samples.write(tmp_path / "bad", samples.RawSamples("b", "amd", 1, 2, (), np.array([5], np.int32),
                                                           np.array([0], np.uint8)))


def test_profile_expansion_bins_back(golden_cases):
    """Every golden profile expands into a raw stream whose binning (numpy,
    the test oracle) reproduces its per-class counts."""
    from paper_2604_20032_b200 import samples
    for ks, pf, cfg, exp in golden_cases["corpus_c1.npz"][:12]:
        rs = samples.from_profile(ks, pf)
        lut = rs.lut()
        cls = np.bincount(rs.pc.astype(np.int64) * 8 + lut[rs.cat], minlength=ks.n_instr * 8)
        assert np.array_equal(cls.reshape(-1, 8), pf.cls_cnt.reshape(-1, 8)), ks.name


@pytest.mark.gpu
def test_file_to_device_session(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle
    from paper_2604_20032_b200 import abi, api, samples, synth
    from paper_2604_20032_b200 import enums as E
    wl = _c2(0.2)
    rs = samples.RawSamples("c2", "amd", wl.profile.period, wl.kernel.n_instr,
                            E.vendor_categories("amd"), wl.pc, wl.cat)
    samples.write(tmp_path / "c2.leosmp", rs)
    back = samples.read(tmp_path / "c2.leosmp")
    sess = api.Session(wl.kernel, wl.profile, back.n_samples, abi.make_config(dialect="amd"))
    sess.stage(wl.kernel, wl.profile, back.pc, back.cat, back.lut())
    r = sess.analyze()
    o = oracle.run(wl.kernel, synth.bin_host(wl), abi.make_config(dialect="amd"))
    assert np.array_equal(r["e_stalled"], o.e_stalled)
    assert np.array_equal(r["e_blame"], o.e_blame)


def test_three_byte_stream_round_trip():
    """device.pack_samples24: little-endian 24-bit words pc << cb | category
    (ABI v4 packed_bytes = 3), 4 category bits (NVIDIA / AMD) or 5 (Intel)."""
    from paper_2604_20032_b200 import device
    from paper_2604_20032_b200 import enums as E
    rng = np.random.default_rng(3)
    for cb, n_instr in ((4, 1 << 20), (5, 1 << 19)):
        n = 1001                                   # not a multiple of 4
        pc = rng.integers(0, n_instr, n).astype(np.int32)
        cat = rng.integers(0, 1 << cb, n).astype(np.uint8)
        b = device.pack_samples24(pc, cat, cb)
        assert b.size % 4 == 0 and b.size >= 3 * n
        w = b[:3 * n].reshape(n, 3).astype(np.uint32)
        w = w[:, 0] | (w[:, 1] << 8) | (w[:, 2] << 16)
        assert np.array_equal(w >> cb, pc) and np.array_equal(w & ((1 << cb) - 1), cat)
        assert device.packable24(pc, cat, n_instr, cb)
        assert not device.packable24(pc, cat, 2 * n_instr, cb)          # pcs would not fit
        bad = cat.copy()
        bad[0] = 1 << cb
        assert not device.packable24(pc, bad, n_instr, cb)
    assert [device.cat_bits_for(len(E.vendor_categories(d))) for d in E.DIALECTS] == [4, 4, 5]
