"""Critical-path time of pipeline prefixes under CUDA graph replay.

LEO_DBG_STOP=s makes leo_analyze end after stage s (1 build incl. binning,
2 prune, 3 incoming CSR, 4 slice; 0 = whole pipeline).  Each prefix is
captured into its own graph and replayed with L2 flushed before every
replay; the differences between consecutive prefixes are the stages' shares
of the step's critical path.

    python tools/stage_times.py [c2|c3|c5] [--reps R] [--scale s]
"""
import argparse
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2604_20032_b200 import abi, device, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c2")
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--stops", default="1,2,3,4,0")
args = ap.parse_args()

dev = torch.device("cuda:0")
wl = synth.config_workload(args.config, scale=args.scale)
dk = device.DeviceKernel(wl.kernel, dev)
dp = device.DeviceProfile(wl.profile, wl.kernel.n_instr, dev)
ds = device.DeviceSamples(wl.pc, wl.cat, wl.lut, dev)
cfg = abi.make_config(dialect=wl.kernel.dialect)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
names = {5: "build + addr branch", 6: "build + prune (no addr)", 1: "bin + build", 2: "+ prune", 3: "+ incoming", 4: "+ slice", 0: "+ blame + lines (full)"}
prev = 0.0
for stop in [int(x) for x in args.stops.split(",")]:
    os.environ["LEO_DBG_STOP"] = str(stop)
    an = device.Analyzer(dk, dev)
    an.run(dp, cfg, ds)
    an.capture(dp, cfg, ds)
    times = []
    for r in range(args.reps + 3):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        an.replay()
        e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            times.append(e0.elapsed_time(e1) * 1e3)
    times.sort()
    med = times[len(times) // 2]
    print(f"{args.config} stop={stop} {names[stop]:24s} median {med:8.1f} us  (+{med - prev:7.1f})  min {times[0]:8.1f}")
    prev = med
    del an
