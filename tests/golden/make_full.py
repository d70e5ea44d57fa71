"""Full-size golden digests: run the REFERENCE (stalltrace) on the BASELINE
configs at full size, here in the authoring container, and store per-field
digests (tests/digest.py) in tests/golden/full_digests.json.

    python tests/golden/make_full.py [c2] [c3] [c5] [c4]

  c2   synthetic AMD, 10,000 instructions, 1 M raw samples binned (seed 2)
  c3   synthetic Intel, 50,000 instructions, 5 M raw samples (seed 3)
  c5   synthetic NVIDIA, 1,000,000 instructions, 100 M raw samples (seed 5)
  c4   C4_SUBSET kernels of the 2,000 x 20,000-instruction batch

Each kernel goes through the reference's own
build_graph -> run_pruning(AnalysisConfig()) -> attribute_blame(pruned,
base_graph=graph) (report.py:132-142), plus the frozen slice / line
restatements (tests/canon.py).  The samples are binned with numpy.bincount
(synth.bin_host), the reference's pre-binned input form.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[2]
sys.path[:0] = [str(REPO), str(REPO / "tests"), str(REPO / "tests" / "golden"), "/root/reference/pkg/src"]

import stalltrace as st  # noqa: E402
from stalltrace import analysis  # noqa: E402

import digest  # noqa: E402
from make_golden import expected_for  # noqa: E402
from paper_2604_20032_b200 import soa, synth  # noqa: E402

OUT = REPO / "tests" / "golden" / "full_digests.json"
C4_SUBSET = (0, 1, 2, 3, 4, 5, 6, 7, 8, 997, 998, 999, 1997, 1998, 1999)


def one(wl, tag):
    t0 = time.time()
    pf = synth.bin_host(wl)
    att = soa.decode_to_reference(wl.kernel, pf, st)
    t1 = time.time()
    _, _, x = expected_for(att, analysis.AnalysisConfig(), ks=wl.kernel, pf=pf)
    t2 = time.time()
    d = digest.digests(x)
    d["_meta"] = {"n_instr": wl.kernel.n_instr, "n_samples": wl.n_samples,
                  "edges": len(x["bprod"]), "pruned": len(x["pprod"]), "entries": len(x["bl_stalled"]),
                  "reference_seconds": round(t2 - t1, 1), "decode_seconds": round(t1 - t0, 1)}
    print(tag, d["_meta"], flush=True)
    return d


def main():
    tags = sys.argv[1:] or ["c2", "c3", "c4", "c5"]
    out = json.loads(OUT.read_text()) if OUT.exists() else {}
    for tag in tags:
        if tag == "c4":
            lines = synth.LineTable(4096, seed=999)
            for k in C4_SUBSET:
                out[f"c4_{k}"] = one(synth.c4_kernel(k, lines), f"c4_{k}")
                OUT.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
        else:
            out[tag] = one(synth.config_workload(tag), tag)
            OUT.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
