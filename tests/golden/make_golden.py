"""Generate tests/golden/*.npz by running the REFERENCE (stalltrace) here.

Run in the authoring container (the reference is importable only here):

    python tests/golden/make_golden.py

Sources of kernels, all pushed through the reference's own
build_graph -> run_pruning -> attribute_blame(pruned, base_graph=graph)
(report.py:132-142):

  1. every AttachedKernel the reference's own test suite builds
     (captured by wrapping stalltrace.depgraph.build_graph while the suite
     runs from a scratch copy of /root/reference/pkg/tests);
  2. the bundled corpus (ltimes_{nvidia,amd,intel}) and the perf-envelope
     generator `_large_kernel(512, 2560)` (C1, test_acceptance.py:402-465);
  3. random_world seeds x 3 dialects and random_cfg_kernel seeds
     (generators.py:85-238) under several AnalysisConfigs;
  4. scaled-down synthetic C2/C3/C5 workloads from paper_2604_20032_b200.synth.

Outputs are stored as arrays (tests/golden_io.py); the oracle and the CUDA
path are compared against them by tests/test_oracle_golden.py and
tests/test_gpu_parity.py.
"""

from __future__ import annotations

import hashlib
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REPO), str(REPO / "tests"), str(REF / "src")]

import stalltrace as st  # noqa: E402
from stalltrace import analysis, depgraph  # noqa: E402

import canon  # noqa: E402
import golden_io  # noqa: E402
from paper_2604_20032_b200 import enums as E  # noqa: E402
from paper_2604_20032_b200 import soa, synth  # noqa: E402

OUT = REPO / "tests" / "golden"


def expected_for(att, cfg, ks=None, pf=None):
    """Reference outputs for one attached kernel, as arrays (`ks` / `pf`: the
    SoA the kernel was decoded from, when the caller has it)."""
    g = depgraph.build_graph(att)
    pr = analysis.run_pruning(g, cfg)
    bl = analysis.attribute_blame(pr, base_graph=g)
    if ks is None:
        ks, pf = soa.encode_attached(att)
    x = {}

    def edge_arrays(edges, prefix):
        prod = np.array([e[0] for e in edges], dtype=np.int32)
        cons = np.array([e[1] for e in edges], dtype=np.int32)
        meta = []
        npaths, first, plen, pacc = [], [], [], []
        for e in edges:
            kind, ref, dc, paths = e[2], e[3], e[4], e[5]
            r27 = 0 if ref is None else (ref[1] | (ref[2] << 16) | (ref[0] << 24))
            meta.append(r27 | (kind << 27) | (dc << 30))
            npaths.append(len(paths))
            first.append(len(plen) if paths else -1)
            for ln, acc in paths:
                plen.append(ln)
                pacc.append(acc)
        x[prefix + "prod"], x[prefix + "cons"] = prod, cons
        x[prefix + "meta"] = np.array(meta, dtype=np.uint32)
        if prefix == "p":
            x["npaths"] = np.array(npaths, dtype=np.int32)
            x["first"] = np.array(first, dtype=np.int32)
            x["plen"] = np.array(plen, dtype=np.int32)
            x["pacc"] = np.array(pacc, dtype=np.float64)

    edge_arrays(canon.ref_edges(g, with_paths=False), "b")
    edge_arrays(canon.ref_edges(pr), "p")
    x["diags"] = np.array(list(pr.diagnostics), dtype=np.str_)
    cb = canon.ref_blame(bl)
    x["bl_stalled"] = np.array([b[0] for b in cb], dtype=np.int32)
    x["bl_cause"] = np.array([-1 if b[1] is None else b[1] for b in cb], dtype=np.int32)
    x["bl_kind"] = np.array([255 if b[2] is None else b[2] for b in cb], dtype=np.uint8)
    x["bl_sub"] = np.array([255 if b[3] is None else b[3] for b in cb], dtype=np.uint8)
    x["bl_blame"] = np.array([b[4] for b in cb], dtype=np.float64)
    x["bl_factors"] = np.array([b[5] if b[5] is not None else (np.nan,) * 4 for b in cb],
                               dtype=np.float64).reshape(-1, 4)
    x["bl_reg"] = np.array(["" if b[6] is None else b[6] for b in cb], dtype=np.str_)
    x["level"] = np.array(canon.ref_slice(pr, att), dtype=np.int32)
    keys = ks.lines
    key_of = lambda i: keys[ks.line_id[i]]  # noqa: E731
    lb, ls = canon.ref_lines(bl, att, key_of)
    pos = {k: i for i, k in enumerate(keys)}
    x["line_blame"] = np.zeros(len(keys), dtype=np.float64)
    x["line_stall"] = np.zeros(len(keys), dtype=np.float64)
    for k, v in lb.items():
        x["line_blame"][pos[k]] = v
    for k, v in ls.items():
        x["line_stall"][pos[k]] = v
    return ks, pf, x


def cfg_dict(cfg, dialect):
    th = None
    if cfg.latency is not None:
        th = E.dense_thresholds((c.value, v) for c, v in cfg.latency.thresholds)
    return dict(stage_mask=list(cfg.stage_mask), prune_exec=bool(cfg.prune_exec),
                max_paths=cfg.max_paths, max_depth=cfg.max_depth, thresholds=th)


def capture_reference_suite():
    """Run the reference test suite from a scratch copy, capturing every
    AttachedKernel handed to build_graph."""
    import pytest
    seen: list = []
    orig = depgraph.build_graph

    def wrapped(attached):
        seen.append(attached)
        return orig(attached)

    depgraph.build_graph = wrapped
    st.build_graph = wrapped
    st.report.build_graph = wrapped
    tmp = Path(tempfile.mkdtemp())
    shutil.copytree(REF / "tests", tmp / "tests")
    try:
        pytest.main([str(tmp / "tests"), "-q", "-x", "-p", "no:cacheprovider",
                     "-k", "not performance_envelope"])
    finally:
        depgraph.build_graph = orig
        st.build_graph = orig
        st.report.build_graph = orig
        shutil.rmtree(tmp, ignore_errors=True)
    return seen


def digest(ks, pf):
    h = hashlib.sha1()
    for f in golden_io.K_FIELDS + ("n_units",):
        h.update(np.ascontiguousarray(getattr(ks, f)).tobytes())
    for f in golden_io.P_FIELDS:
        h.update(np.ascontiguousarray(getattr(pf, f)).tobytes())
    h.update(str(pf.period).encode())
    return h.hexdigest()


def add(cases, seen, att, cfg, tag):
    ks, pf = soa.encode_attached(att)
    key = (digest(ks, pf), repr(cfg_dict(cfg, ks.dialect)))
    if key in seen:
        return
    seen.add(key)
    ks, pf, x = expected_for(att, cfg)
    ks.name = f"{tag}:{ks.name}"
    cases.append(golden_io.pack_case(ks, pf, cfg_dict(cfg, ks.dialect), x))


def main():
    # 1. reference suite kernels (run first: the suite imports its own
    #    generators/conftest modules from the scratch copy)
    suite = capture_reference_suite()
    for name in list(sys.modules):
        if name in ("generators", "oracles", "conftest") or name.startswith("test_"):
            del sys.modules[name]
    sys.path[:] = [p for p in sys.path if "/tmp/" not in p]
    sys.path.insert(0, str(REF / "tests"))
    import generators
    from test_acceptance import _large_kernel

    default = analysis.AnalysisConfig()
    variants = [
        analysis.AnalysisConfig(prune_exec=True),
        analysis.AnalysisConfig(stage_mask=()),
        analysis.AnalysisConfig(stage_mask=(1, 2), prune_exec=True),
        analysis.AnalysisConfig(max_paths=2, max_depth=6),
        analysis.AnalysisConfig(stage_mask=(3,), max_paths=3, max_depth=5),
    ]

    cases, seen = [], set()
    for att in suite:
        add(cases, seen, att, default, "suite")
    golden_io.save(OUT / "reference_suite.npz", cases)
    print("reference_suite:", len(cases))

    # 2. corpus + C1
    cases, seen = [], set()
    corpus = REF / "tests" / "corpus"
    for v in ("nvidia", "amd", "intel"):
        d = st.Dialect.from_name(v)
        cfg = st.parse_kernels(d, (corpus / f"ltimes_{v}.s").read_text())["ltimes_noview"]
        prof = st.load_profile((corpus / f"ltimes_{v}.prof").read_text())
        att = st.attach(cfg, prof)
        for c in [default] + variants:
            add(cases, seen, att, c, f"corpus_{v}")
    cfg, prof = _large_kernel(512, 2560)
    att = st.attach(cfg, prof)
    for c in [default] + variants:
        add(cases, seen, att, c, "c1_large512")
    golden_io.save(OUT / "corpus_c1.npz", cases)
    print("corpus_c1:", len(cases))

    # 3. random worlds / random CFG kernels
    cases, seen = [], set()
    for v in ("nvidia", "amd", "intel"):
        for s in range(100):
            att = generators.random_world(s, st.Dialect(v))
            add(cases, seen, att, default, f"world_{v}")
            add(cases, seen, att, variants[s % len(variants)], f"world_{v}")
    for s in range(80):
        cfgk = generators.random_cfg_kernel(s)
        prof = st.profile.KernelProfile(kernel_name=cfgk.kernel_name, dialect=cfgk.dialect,
                                        sampling_period_cycles=10, samples=())
        add(cases, seen, st.attach(cfgk, prof), default, "cfg")
    golden_io.save(OUT / "random.npz", cases)
    print("random:", len(cases))

    # 4. scaled synthetic configs (kernel + binned raw samples)
    cases, seen = [], set()
    for tag, scale in (("c2", 0.05), ("c2", 0.2), ("c3", 0.02), ("c3", 0.06), ("c5", 0.001),
                       ("c5", 0.004)):
        wl = synth.config_workload(tag, scale=scale)
        ks = wl.kernel
        # restrict the line table to the lines this kernel uses (fixture size)
        used = np.unique(ks.line_id)
        remap = np.full(len(ks.lines), -1, dtype=np.int64)
        remap[used] = np.arange(used.shape[0])
        ks.lines = [ks.lines[int(u)] for u in used]
        ks.line_id = remap[ks.line_id].astype(np.int32)
        pf = synth.bin_host(wl)
        att = soa.decode_to_reference(ks, pf, st)
        for c in (default, variants[0]):
            add(cases, seen, att, c, f"synth_{tag}_{scale}")
    golden_io.save(OUT / "synth.npz", cases)
    print("synth:", len(cases))


if __name__ == "__main__":
    main()
