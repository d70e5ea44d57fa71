"""Generate tests/golden/reports.npz by running the REFERENCE's build_report +
render_text / render_structured (report.py:128-346) here.

    python tests/golden/make_reports.py

Cases: the bundled corpus (ltimes_{nvidia,amd,intel}, checked against the
committed corpus/*.report.{txt,json} first), `_large_kernel(512, 2560)`
(C1), random_world kernels of the three dialects and a scaled synthetic C2
kernel, each under a few (top_n, include_unsampled, chain_depth, config)
settings.  Every case stores the kernel / profile SoA, the host report
metadata (mnemonics, offsets, source locations, latency-table echo) and the
two expected renderings.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REPO), str(REF / "tests"), str(REPO / "tests"), str(REF / "src")]

import stalltrace as st  # noqa: E402
from stalltrace import analysis, report  # noqa: E402

import golden_io  # noqa: E402
from paper_2604_20032_b200 import enums as E  # noqa: E402
from paper_2604_20032_b200 import soa, synth  # noqa: E402

OUT = REPO / "tests" / "golden" / "reports.npz"


def cfg_dict(cfg, dialect):
    """AnalysisConfig -> fixture dict (same layout as make_golden.py)."""
    th = None
    if cfg.latency is not None:
        th = E.dense_thresholds((c.value, v) for c, v in cfg.latency.thresholds)
    return dict(stage_mask=list(cfg.stage_mask), prune_exec=bool(cfg.prune_exec),
                max_paths=cfg.max_paths, max_depth=cfg.max_depth, thresholds=th)
NONE = "\x00"


def case(cfg, prof, config, tag, top_n=10, include_unsampled=False, chain_depth=32):
    rep = report.build_report(cfg, prof, config, top_n=top_n, include_unsampled=include_unsampled,
                              chain_depth=chain_depth)
    att = st.attach(cfg, prof)
    ks, pf = soa.encode_attached(att)
    ks.name = f"{tag}:{ks.name}"
    table = config.table_for(cfg.dialect)
    rmeta = dict(kernel_name=cfg.kernel_name, vendor=cfg.dialect.value,
                 period=prof.sampling_period_cycles, top_n=top_n,
                 include_unsampled=include_unsampled, chain_depth=chain_depth,
                 echo=dict(stage_mask=list(config.stage_mask), prune_exec=config.prune_exec,
                           max_paths=config.max_paths, max_depth=config.max_depth,
                           latency_units=table.units,
                           latency_table=[[c.value, v] for c, v in
                                          sorted(table.thresholds, key=lambda kv: kv[0].value)]))
    x = {"text": np.array([report.render_text(rep)]),
         "json": np.array([report.render_structured(rep)]),
         "rmeta": np.array([json.dumps(rmeta)]),
         "mnemonics": np.array([i.mnemonic for i in cfg.instructions], dtype=np.str_),
         "srclocs": np.array([str(i.src_loc) if i.src_loc else NONE for i in cfg.instructions],
                             dtype=np.str_)}
    return golden_io.pack_case(ks, pf, cfg_dict(config, ks.dialect), x)


def main():
    import generators
    from test_acceptance import _large_kernel

    default = analysis.AnalysisConfig()
    cases = []
    corpus = REF / "tests" / "corpus"
    for v in ("nvidia", "amd", "intel"):
        d = st.Dialect.from_name(v)
        cfg = st.parse_kernels(d, (corpus / f"ltimes_{v}.s").read_text())["ltimes_noview"]
        prof = st.load_profile((corpus / f"ltimes_{v}.prof").read_text())
        rep = report.build_report(cfg, prof, default)
        assert report.render_text(rep) == (corpus / f"ltimes_{v}.report.txt").read_text()
        assert report.render_structured(rep) == (corpus / f"ltimes_{v}.report.json").read_text()
        cases.append(case(cfg, prof, default, f"corpus_{v}"))
        cases.append(case(cfg, prof, default, f"corpus_{v}", top_n=2, include_unsampled=True,
                          chain_depth=2))
        cases.append(case(cfg, prof, analysis.AnalysisConfig(stage_mask=()), f"corpus_{v}",
                          top_n=20, include_unsampled=True))
    cfg, prof = _large_kernel(512, 2560)
    cases.append(case(cfg, prof, default, "c1_large512", top_n=25))
    cases.append(case(cfg, prof, analysis.AnalysisConfig(prune_exec=True, max_paths=3),
                      "c1_large512", top_n=40, include_unsampled=True, chain_depth=5))
    for v in ("nvidia", "amd", "intel"):
        for s in range(25):
            att = generators.random_world(s, st.Dialect(v))
            cases.append(case(att.cfg, att.profile, default, f"world_{v}", top_n=5 + s % 7,
                              include_unsampled=bool(s % 3 == 0), chain_depth=3 + s % 30))
    wl = synth.config_workload("c2", scale=0.05)
    sk = soa.decode_to_reference(wl.kernel, synth.bin_host(wl), st)
    cases.append(case(sk.cfg, sk.profile, default, "synth_c2", top_n=50))
    golden_io.save(OUT, cases)
    print("reports:", len(cases))


if __name__ == "__main__":
    main()
