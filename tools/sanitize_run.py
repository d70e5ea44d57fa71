"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): the three corpus kernels from the golden vectors and
synthetic C2 / C3 / C5 kernels at reduced scale with raw samples, eager
launches through the C ABI, each checked against the oracle.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [--quick] [--big] [--packed3]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import golden_io  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2604_20032_b200 import abi, device, synth  # noqa: E402

dev = torch.device("cuda:0")
quick = "--quick" in sys.argv
cases = golden_io.load(ROOT / "tests" / "golden" / "corpus_c1.npz")
picked, seen = [], set()
for c in cases:                       # one case per corpus kernel (nvidia / amd / intel)
    if c[0].name not in seen:
        seen.add(c[0].name)
        picked.append(c)
for ks, pf, cfg, exp in picked:
    r = device.analyze_soa(ks, pf, golden_io.config_of(cfg, ks.dialect), device=dev)
    assert np.array_equal(r["bprod"], exp["bprod"]) and np.array_equal(r["pprod"], exp["pprod"]), ks.name
    print("corpus", ks.name, "ok", flush=True)
# --big adds C5 at a quarter (12.5 k blocks: the tier-1 reach search, the one-pass
# hashed binning of 25 M samples, the big-kernel sync / prune tiers)
runs = (("c2", 0.1), ("c3", 0.02), ("c5", 0.002)) if quick else (("c2", 0.2), ("c3", 0.05), ("c5", 0.005))
if "--big" in sys.argv:
    runs += (("c5", 0.25),)
for tag, scale in runs:
    wl = synth.config_workload(tag, scale=scale)
    r = device.analyze_soa(wl.kernel, wl.profile, abi.make_config(dialect=wl.kernel.dialect),
                           samples=(wl.pc, wl.cat, wl.lut), device=dev)
    o = oracle.run(wl.kernel, synth.bin_host(wl))
    for a, b in (("bprod", "prod"), ("bmeta", "meta"), ("pprod", "p_prod"), ("e_blame", "e_blame"),
                 ("level", "level")):
        assert np.array_equal(r[a], getattr(o, b)), (tag, a)
    print(tag, scale, wl.kernel.n_instr, "instrs ok", flush=True)
# --packed3: the 3-byte sample stream (4 and 5 category bits) through the
# one-pass binning, cut to lengths that leave partial 16-sample groups
if "--packed3" in sys.argv:
    for tag, scale in (("c5", 0.05), ("c3", 1.0)):
        wl = synth.config_workload(tag, scale=scale)
        cfg = abi.make_config(dialect=wl.kernel.dialect)
        for cut in (0, 5, 27):
            n = len(wl.pc) - cut
            smp = (wl.pc[:n], wl.cat[:n], wl.lut)
            a = device.analyze_soa(wl.kernel, wl.profile, cfg, samples=smp, device=dev, packed=True, width=3)
            b = device.analyze_soa(wl.kernel, wl.profile, cfg, samples=smp, device=dev, packed=False)
            for key in ("lat", "cls_cnt", "e_blame"):
                assert np.array_equal(a[key], b[key]), (tag, cut, key)
        print(tag, "3-byte stream ok", flush=True)
print("sanitize_run ok")
