"""Golden vectors for the dataflow sub-steps of build_graph, made by running
the REFERENCE here:

    python tests/golden/make_dataflow.py   ->  tests/golden/dataflow.npz

Per kernel (the corpus, random_cfg_kernel seeds and random_world kernels of
the reference's generators.py, a scaled synthetic C2/C3/C5 kernel each):

  reaching_definitions(cfg) (depgraph.py:135-177) as a CSR over (block, dense
      unit id) pairs with sorted def sets: x_reach_off[B*U+1], x_reach_defs
  per_use_link(cfg, reach_in) (depgraph.py:188-223) as a sorted link set:
      x_link_prod / x_link_cons / x_link_meta (ref27 | kind << 27)
  liveness_filter(cfg, links) (depgraph.py:274-293) on the pipeline's links
      plus random cross-block candidates (some dead): x_lf_prod / x_lf_cons /
      x_lf_meta and the reference's verdict x_lf_keep

Stored with tests/golden_io.py (kernel SoA + expected arrays).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REPO), str(REPO / "tests"), str(REF / "src"), str(REF / "tests")]

import stalltrace as st  # noqa: E402
from stalltrace import depgraph  # noqa: E402

import golden_io  # noqa: E402
from paper_2604_20032_b200 import enums as E  # noqa: E402
from paper_2604_20032_b200 import soa, synth  # noqa: E402

OUT = REPO / "tests" / "golden" / "dataflow.npz"


def ref27(ref):
    return ref.index | (ref.span << 16) | (E.RC_IDX[ref.reg_class.value] << 24)


def expected(cfg, ks, rng):
    U, B = ks.n_units, ks.n_blocks
    base = np.asarray(ks.unit_base, dtype=np.int64)
    uid = lambda unit: int(base[E.RC_IDX[unit[0].value]]) + unit[1]  # noqa: E731
    reach = depgraph.reaching_definitions(cfg)
    off = np.zeros(B * U + 1, dtype=np.int32)
    sets = {}
    for b, d in enumerate(reach):
        for unit, defs in d.items():
            sets[b * U + uid(unit)] = sorted(defs)
    defs_flat = []
    for x in range(B * U):
        s = sets.get(x, ())
        defs_flat.extend(s)
        off[x + 1] = len(defs_flat)
    links, _ = depgraph.per_use_link(cfg, reach)
    lk = sorted({(l.producer, l.consumer, ref27(l.register) | (E.EK_IDX[l.kind.value] << 27)) for l in links})
    # liveness_filter candidates: the pipeline's links + random cross-block ones
    cand = list(links)
    instrs = cfg.instructions
    users = [i for i, ins in enumerate(instrs) if ins.srcs]
    defs_ = [i for i, ins in enumerate(instrs) if ins.dests]
    for _ in range(min(200, 4 * len(instrs))):
        if not users or not defs_:
            break
        c = users[rng.integers(len(users))]
        p = defs_[rng.integers(len(defs_))]
        r = instrs[c].srcs[rng.integers(len(instrs[c].srcs))]
        cand.append(depgraph.UseLink(producer=p, consumer=c, register=r, kind=depgraph.EdgeKind.RAW))
    kept = set(id(l) for l in depgraph.liveness_filter(cfg, cand))
    x = dict(reach_off=off, reach_defs=np.asarray(defs_flat, dtype=np.int32),
             link_prod=np.array([t[0] for t in lk], np.int32), link_cons=np.array([t[1] for t in lk], np.int32),
             link_meta=np.array([t[2] for t in lk], np.uint32),
             lf_prod=np.array([l.producer for l in cand], np.int32),
             lf_cons=np.array([l.consumer for l in cand], np.int32),
             lf_meta=np.array([ref27(l.register) | (E.EK_IDX[l.kind.value] << 27) for l in cand], np.uint32),
             lf_keep=np.array([1 if id(l) in kept else 0 for l in cand], np.uint8))
    return x


def main():
    import generators
    rng = np.random.default_rng(11)
    cases = []
    cfgs = []
    corpus = REF / "tests" / "corpus"
    for v in ("nvidia", "amd", "intel"):
        d = st.Dialect.from_name(v)
        cfgs.append(st.parse_kernels(d, (corpus / f"ltimes_{v}.s").read_text())["ltimes_noview"])
    for s in range(120):
        cfgs.append(generators.random_cfg_kernel(s))
    for s in range(60):
        cfgs.append(generators.random_world(500 + s, st.Dialect(("nvidia", "amd", "intel")[s % 3])).cfg)
    for tag, scale in (("c2", 0.1), ("c3", 0.03), ("c5", 0.002)):
        wl = synth.config_workload(tag, scale=scale)
        cfgs.append(soa.decode_to_reference(wl.kernel, None, st))
    for cfg in cfgs:
        ks = soa.encode_cfg(cfg)
        pf = soa.ProfileSoA(period=1, lat=np.zeros(ks.n_instr, np.int32),
                            cls_cnt=np.zeros((ks.n_instr, 8), np.int32),
                            exec_cnt=np.full(ks.n_instr, -1, np.int64),
                            total=np.full(ks.n_instr, -1, np.int32), eff=np.ones(ks.n_instr),
                            sampled=np.zeros(ks.n_instr, np.uint8))
        cases.append(golden_io.pack_case(ks, pf, {"stage_mask": [], "prune_exec": False, "max_paths": 64,
                                                 "max_depth": 512, "thresholds": None},
                                         expected(cfg, ks, rng)))
    golden_io.save(OUT, cases)
    print("dataflow:", len(cases))


if __name__ == "__main__":
    main()
