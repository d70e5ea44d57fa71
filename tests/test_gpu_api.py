"""GPU parity of the stand-alone C-ABI entry points behind the drop-in API
(ops.py -> leo_prune / leo_blame / leo_slice / leo_self_blame / leo_coverage /
leo_rank_hotspots / leo_trace_chain / leo_line_rollup /
leo_reaching_definitions / leo_liveness_filter), on the reference's golden
vectors, with edge lists in ARBITRARY order (LeoEdges.n_regular = NULL: the
reference's DependencyGraph holds any edge tuple) and stages CHAINED one at a
time with valid_paths carried (analysis.py:143-314), the two call patterns
the fused pipeline never sees."""

import numpy as np
import pytest

import golden_io
from conftest import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASE_FILES = ("corpus_c1.npz", "random.npz", "reference_suite.npz")


@pytest.fixture(scope="module")
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_20032_b200 import _lib
    _lib.lib()
    return torch.device("cuda:0")


@pytest.fixture(scope="module")
def cases(golden_cases):
    out = []
    for f in CASE_FILES:
        out += golden_cases[f]
    return out


def kern(ks, pf, dev):
    from paper_2604_20032_b200 import device
    return device.DeviceKernel(ks, dev), device.DeviceProfile(pf, ks.n_instr, dev)


def key(p, c, m):
    return (int(p), int(c), int(m))


def golden_paths(exp, x):
    n = int(exp["npaths"][x])
    f = int(exp["first"][x])
    return tuple(zip(exp["plen"][f:f + n].tolist(), exp["pacc"][f:f + n].tolist())) if n else ()


def got_paths(r, x):
    n = int(r["npaths"][x])
    f = int(r["first"][x])
    return tuple(zip(r["plen"][f:f + n].tolist(), r["pacc"][f:f + n].tolist())) if n else ()


def path_diags(exp):
    return [str(s) for s in exp["diags"] if str(s).startswith("path enumeration capped")]


def test_prune_arbitrary_order_and_chained_stages(cases, cuda):
    from paper_2604_20032_b200 import diagnostics, ops
    rng = np.random.default_rng(5)
    bad = []
    for ks, pf, cfg, exp in cases:
        dk, dp = kern(ks, pf, cuda)
        bp, bc, bm = exp["bprod"], exp["bcons"], exp["bmeta"].astype(np.uint32)
        pk = {key(p, c, m): x for x, (p, c, m) in enumerate(zip(exp["pprod"], exp["pcons"], exp["pmeta"]))}
        lcfg = golden_io.config_of(cfg, ks.dialect)
        # (1) one call over the base edges in a random order
        perm = rng.permutation(len(bp))
        d = ops.DevEdges.from_arrays(cuda, bp[perm], bc[perm], bm[perm])
        r, _ = ops.prune(dk, dp, lcfg, d)
        want = [x for x in perm if key(bp[x], bc[x], bm[x]) in pk]
        got = list(zip(r["pprod"].tolist(), r["pcons"].tolist(), r["pmeta"].tolist()))
        if got != [key(bp[x], bc[x], bm[x]) for x in want]:
            bad.append((ks.name, "shuffled edge list"))
            continue
        for y, x in enumerate(want):
            if got_paths(r, y) != golden_paths(exp, pk[key(bp[x], bc[x], bm[x])]):
                bad.append((ks.name, "shuffled valid_paths"))
                break
        # (2) the stages one at a time, valid_paths carried from call to call
        d = ops.DevEdges.from_arrays(cuda, bp, bc, bm)
        cur = list(zip(bp.tolist(), bc.tolist(), bm.tolist()))
        diags, r = [], None
        for s in (1, 2, 3, 4):
            if s not in cfg["stage_mask"] or (s == 2 and ks.dialect != "nvidia") or (s == 4 and not cfg["prune_exec"]):
                continue
            one = golden_io.config_of(dict(cfg, stage_mask=[s]), ks.dialect)
            r, d = ops.prune(dk, dp, one, d)
            cur = list(zip(r["pprod"].tolist(), r["pcons"].tolist(), r["pmeta"].tolist()))
            diags += diagnostics.render(ks.dialect, ks.offset, r["diag_records"], ordered=True)
        if cur != [key(p, c, m) for p, c, m in zip(exp["pprod"], exp["pcons"], exp["pmeta"])]:
            bad.append((ks.name, "chained stages"))
            continue
        if r is not None and any(got_paths(r, y) != golden_paths(exp, y) for y in range(len(cur))):
            bad.append((ks.name, "chained valid_paths"))
            continue
        if diags != path_diags(exp):
            bad.append((ks.name, "chained diagnostics"))
        # (3) stage 3 again on its own output keeps every edge and its paths (idempotent)
        if r is not None and list(cfg["stage_mask"]) == [3]:
            r2, _ = ops.prune(dk, dp, lcfg, d)
            if not np.array_equal(r2["pprod"], r["pprod"]) or \
                    any(got_paths(r2, y) != got_paths(r, y) for y in range(len(r["pprod"]))):
                bad.append((ks.name, "stage 3 not idempotent"))
    assert not bad, f"{len(bad)} cases differ; first {bad[:5]}"


def test_blame_slice_self_on_arbitrary_order_graphs(cases, cuda):
    from paper_2604_20032_b200 import ops
    rng = np.random.default_rng(9)
    bad = []
    for ks, pf, cfg, exp in cases:
        dk, dp = kern(ks, pf, cuda)
        pp, pc, pm = exp["pprod"], exp["pcons"], exp["pmeta"].astype(np.uint32)
        npaths, first = exp["npaths"], exp["first"]
        base = ops.DevEdges.from_arrays(cuda, exp["bprod"], exp["bcons"], exp["bmeta"])
        # identity order through the arbitrary-order path: bit-exact entries
        d = ops.DevEdges.from_arrays(cuda, pp, pc, pm, npaths, first, exp["plen"], exp["pacc"])
        r = ops.blame(dk, dp, d, base)
        cause = np.where(r["e_edge"] < 0, -1, pp[np.maximum(r["e_edge"], 0)] if len(pp) else -1)
        if not (np.array_equal(r["e_stalled"], exp["bl_stalled"]) and np.array_equal(cause, exp["bl_cause"])
                and np.array_equal(r["e_blame"], exp["bl_blame"])):
            bad.append((ks.name, "blame (list order)"))
            continue
        sub = np.where(r["e_edge"] < 0, r["e_sub"], 255)
        if not np.array_equal(sub.astype(np.uint8), exp["bl_sub"]):
            bad.append((ks.name, "self-blame subcategory"))
            continue
        # shuffled pruned edges: same entries per stalled instruction (blame
        # within 1e-12: the normaliser's summation order follows the list)
        perm = rng.permutation(len(pp))
        inv_first = first[perm] if len(pp) else first
        d2 = ops.DevEdges.from_arrays(cuda, pp[perm], pc[perm], pm[perm], npaths[perm], inv_first,
                                      exp["plen"], exp["pacc"])
        r2 = ops.blame(dk, dp, d2, base)
        c2 = np.where(r2["e_edge"] < 0, -1, pp[perm][np.maximum(r2["e_edge"], 0)] if len(pp) else -1)
        a = sorted(zip(exp["bl_stalled"].tolist(), exp["bl_cause"].tolist(), exp["bl_blame"].tolist()))
        b = sorted(zip(r2["e_stalled"].tolist(), c2.tolist(), r2["e_blame"].tolist()))
        if [x[:2] for x in a] != [x[:2] for x in b] or \
                not np.allclose([x[2] for x in a], [x[2] for x in b], rtol=1e-12, atol=0):
            bad.append((ks.name, "blame (shuffled)"))
            continue
        if not np.array_equal(ops.slice_levels(dk, dp, d2), exp["level"]):
            bad.append((ks.name, "slice (shuffled)"))
            continue
        # self_blame of EVERY instruction; the golden's self entries must agree
        s_sub, s_cyc = ops.self_blame(dk, dp, base, np.arange(ks.n_instr))
        selfs = exp["bl_cause"] < 0
        j = exp["bl_stalled"][selfs]
        if not (np.array_equal(s_sub[j], exp["bl_sub"][selfs]) and
                np.array_equal(s_cyc, pf.lat.astype(np.float64) * pf.period)):
            bad.append((ks.name, "self_blame"))
            continue
        # per-line rollup of the golden entry list
        lb, ls = ops.line_rollup(dk, dp, exp["bl_stalled"], exp["bl_cause"], exp["bl_blame"])
        if not (np.allclose(lb, exp["line_blame"], rtol=1e-9, atol=1e-9) and
                np.allclose(ls, exp["line_stall"], rtol=1e-9, atol=1e-9)):
            bad.append((ks.name, "line rollup"))
    assert not bad, f"{len(bad)} cases differ; first {bad[:5]}"


def chain_restated(stalled, cause, blame, offsets, lat, start, max_depth):
    """trace_chain (analysis.py:499-538) restated over arrays (test side)."""
    by = {}
    for x, s in enumerate(stalled):
        by.setdefault(int(s), []).append(x)
    nodes, ents, visited, node, self_e = [start], [-1], {start}, start, -1
    while len(nodes) < max_depth:
        es = by.get(node)
        if not es:
            break
        best = min(es, key=lambda x: (-blame[x], offsets[cause[x]] if cause[x] >= 0 else float("inf")))
        if cause[best] < 0:
            self_e = best
            break
        if cause[best] in visited:
            break
        nodes.append(int(cause[best]))
        ents.append(best)
        visited.add(int(cause[best]))
        node = int(cause[best])
    return nodes, ents, self_e


def test_coverage_rank_chain(cases, cuda):
    from paper_2604_20032_b200 import ops
    rng = np.random.default_rng(3)
    bad = []
    for ks, pf, cfg, exp in cases[:600]:
        dk, dp = kern(ks, pf, cuda)
        pc, pm = exp["pcons"], exp["pmeta"].astype(np.uint32)
        d = ops.DevEdges.from_arrays(cuda, exp["pprod"], pc, pm)
        nodes, qual = ops.coverage(dk, d)
        cls = {}
        for c, m in zip(pc.tolist(), pm.tolist()):
            cls.setdefault(c, []).append(m >> 30)
        q = sum(1 for v in cls.values() if len(set(v)) in (1, len(v)))
        if (nodes, qual) != (len(cls), q):
            bad.append((ks.name, "coverage"))
            continue
        lat = pf.lat.astype(np.int64)
        for inc in (False, True):
            top = int(rng.integers(1, 12))
            st = sorted(np.flatnonzero(lat > 0).tolist(), key=lambda i: (-lat[i], ks.offset[i]))
            want = (st + (np.flatnonzero(lat == 0).tolist() if inc else []))[:top]
            if ops.rank_hotspots(dk, dp, top, inc) != want:
                bad.append((ks.name, "rank_hotspots"))
        stalled, cause, blame = exp["bl_stalled"], exp["bl_cause"], exp["bl_blame"]
        if len(stalled):
            perm = rng.permutation(len(stalled))          # any entry order
            s, c, b = stalled[perm], cause[perm], blame[perm]
            for start in set(s[:3].tolist()) | {0}:
                for depth in (2, 32):
                    n1, e1, s1 = ops.trace_chain(dk, s, c, b, start, depth)
                    n2, e2, s2 = chain_restated(s, c, b.tolist(), ks.offset, lat, start, depth)
                    if (n1, e1, s1) != (n2, e2, s2):
                        bad.append((ks.name, "trace_chain", start, depth))
    assert not bad, f"{len(bad)} differ; first {bad[:5]}"


def test_dataflow_substeps_match_reference(golden_cases, cuda):
    """reaching_definitions, per_use_link and liveness_filter (depgraph.py:135-293)
    against the reference's outputs (tests/golden/dataflow.npz)."""
    from paper_2604_20032_b200 import ops
    cases = golden_io.load(GOLDEN / "dataflow.npz")
    bad = []
    for ks, pf, cfg, x in cases:
        dk, dp = kern(ks, pf, cuda)
        off, defs = ops.reach_in(dk)
        P = len(off) - 1
        if P != len(x["reach_off"]) - 1:
            bad.append((ks.name, "reach pairs"))
            continue
        # (a set may list a def twice: two blocks of one fallthrough run share their nearest def)
        got = [sorted(set(defs[off[i]:off[i + 1]].tolist())) for i in range(P)]
        want = [x["reach_defs"][x["reach_off"][i]:x["reach_off"][i + 1]].tolist() for i in range(P)]
        if got != want:
            bad.append((ks.name, "reach sets"))
            continue
        b = ops.build(dk)
        r = b["n_regular"]
        links = sorted(zip(b["bprod"][:r].tolist(), b["bcons"][:r].tolist(),
                           (b["bmeta"][:r] & np.uint32(0x3FFFFFFF)).tolist()))
        want = list(zip(x["link_prod"].tolist(), x["link_cons"].tolist(), x["link_meta"].tolist()))
        if links != want:
            bad.append((ks.name, "per_use_link"))
            continue
        keep = ops.liveness_filter(dk, x["lf_prod"], x["lf_cons"], x["lf_meta"])
        if not np.array_equal(keep, x["lf_keep"]):
            bad.append((ks.name, "liveness_filter"))
    assert not bad, f"{len(bad)}/{len(cases)} differ; first {bad[:5]}"


def test_sample_pc_out_of_range_is_an_error(cuda):
    """a raw sample whose pc is outside the kernel is reported
    (LEO_ST_BAD_INPUT -> ValueError), not dropped silently."""
    from paper_2604_20032_b200 import abi, device, synth
    wl = synth.config_workload("c2", scale=0.05)
    pc = wl.pc.copy()
    pc[17] = wl.kernel.n_instr + 5
    with pytest.raises(ValueError, match="sample pc out of range"):
        device.analyze_soa(wl.kernel, wl.profile, abi.make_config(dialect="amd"),
                           samples=(pc, wl.cat, wl.lut), device=cuda)
