"""Report assembly against the reference's reports.

Golden cases: tests/golden/reports.npz (tests/golden/make_reports.py runs the
reference's build_report + render_text / render_structured; the three corpus
kernels are first checked against the committed corpus/*.report.{txt,json}).

  * CPU: the renderers are byte-identical on every golden report (parsed back
    from its structured form);
  * GPU: build_report on the device (analysis + coverage + ranking + cause
    order + trace_chain) renders byte-identical text and JSON.
"""

import json

import numpy as np
import pytest

import golden_io

GOLD = "reports.npz"


@pytest.fixture(scope="module")
def report_cases():
    from conftest import GOLDEN
    return golden_io.load(GOLDEN / GOLD)


def test_renderers_byte_exact(report_cases):
    from paper_2604_20032_b200 import report
    assert len(report_cases) >= 80
    for ks, pf, cfg, exp in report_cases:
        text, js = str(exp["text"][0]), str(exp["json"][0])
        rep = report.parse_structured(js)
        assert report.render_structured(rep) == js, ks.name
        assert report.render_text(rep) == text, ks.name


def test_coverage_and_conservation_helpers():
    from paper_2604_20032_b200 import report
    assert report._coverage(0, 0) == (1.0, True)
    assert report._coverage(4, 3) == (0.75, False)
    lat = np.array([2, 0, 1], dtype=np.int32)
    report.check_conservation(lat, 10, np.array([0, 0, 2]), np.array([5.0, 15.0, 10.0]))
    with pytest.raises(report.InternalInvariantError):
        report.check_conservation(lat, 10, np.array([0, 2]), np.array([19.0, 10.0]))


@pytest.mark.gpu
def test_device_report_matches_reference(report_cases):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_20032_b200 import api, report
    bad = []
    for ks, pf, cfg, exp in report_cases:
        rmeta = json.loads(str(exp["rmeta"][0]))
        meta = report.meta_from_fixture(rmeta, exp["mnemonics"], exp["srclocs"])
        rep = api.build_report_soa(ks, pf, golden_io.config_of(cfg, ks.dialect), meta,
                                   top_n=rmeta["top_n"], include_unsampled=rmeta["include_unsampled"],
                                   chain_depth=rmeta["chain_depth"])
        for kind, got, want in (("json", report.render_structured(rep), str(exp["json"][0])),
                                ("text", report.render_text(rep), str(exp["text"][0]))):
            if got != want:
                i = next((x for x, (p, q) in enumerate(zip(got, want)) if p != q), min(len(got), len(want)))
                bad.append((ks.name, kind, got[max(0, i - 80):i + 40], want[max(0, i - 80):i + 40]))
    assert not bad, f"{len(bad)} report renderings differ: {bad[:5]}"


@pytest.mark.gpu
def test_listing_text_to_report_end_to_end(report_cases):
    """Listing text -> native front-end -> device analysis + report assembly
    -> rendered report, byte-identical to the reference's corpus reports
    (profile SoA from the golden fixture: profile JSON loading stays on the
    reference side)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from conftest import GOLDEN
    from paper_2604_20032_b200 import api, front, report
    z = np.load(GOLDEN / "front.npz")
    fcases, tables = json.loads(str(z["cases"])), json.loads(str(z["tables"]))
    checked = 0
    for ks_ref, pf, cfg, exp in report_cases:
        if not ks_ref.name.startswith("corpus_"):
            continue
        d = ks_ref.dialect
        text = next(c["text"] for c in fcases if c["dialect"] == d and "ltimes_noview" in c["text"][:400])
        ks, meta = front.parse_kernels_soa(d, text, tables[d])["ltimes_noview"]
        rmeta = json.loads(str(exp["rmeta"][0]))
        rm = report.meta_from_fixture(rmeta, meta["mnemonics"],
                                      [s if s is not None else "" for s in meta["src_locs"]])
        ks.prefix_diagnostics = ks_ref.prefix_diagnostics       # attach diagnostics (profile side)
        rep = api.build_report_soa(ks, pf, golden_io.config_of(cfg, d), rm, top_n=rmeta["top_n"],
                                   include_unsampled=rmeta["include_unsampled"],
                                   chain_depth=rmeta["chain_depth"])
        assert report.render_text(rep) == str(exp["text"][0]), ks_ref.name
        assert report.render_structured(rep) == str(exp["json"][0]), ks_ref.name
        checked += 1
    assert checked == 9
