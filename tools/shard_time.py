"""Device time of one rank's share of C5 under stalled-PC sharding (world W,
rank r), one GPU, graph replay: what each GPU of a W-GPU run does.

    python tools/shard_time.py <rank> [world]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_20032_b200 import abi, device, synth  # noqa: E402
from paper_2604_20032_b200 import dist as D  # noqa: E402

rank = int(sys.argv[1])
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dev = torch.device("cuda:0")
wl = synth.config_workload("c5")
(lo, hi), pc, cat = D.shard_workload(wl, rank, world)
dk = device.DeviceKernel(wl.kernel, dev)
dp = device.DeviceProfile(wl.profile, wl.kernel.n_instr, dev)
ds = device.DeviceSamples(pc, cat, wl.lut, dev)
an = device.Analyzer(dk, dev, do_slice=False)
cfg = abi.make_config(dialect="nvidia", consumer_range=(lo, hi))
an.run(dp, cfg, ds)
an.capture(dp, cfg, ds)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ts = []
for s in range(23):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    an.replay()
    b.record()
    torch.cuda.synchronize()
    if s >= 3:
        ts.append(a.elapsed_time(b))
print(f"c5 rank {rank}/{world} consumers [{lo}, {hi}) samples {len(pc)}: {np.median(ts) * 1e3:.1f} us per step")

if "--timeline" in sys.argv:
    tr = device.Tracer(capacity=4096, timeline=True)
    an.set_tracer(tr)
    an.capture(dp, cfg, ds, trace_in_graph=True)
    for _ in range(3):
        flush.zero_()
        torch.cuda.synchronize()
        torch.cuda._sleep(20_000_000)
        an.replay()
        torch.cuda.synchronize()
    tl = tr.timeline()
    an.set_tracer(None)
    end = max(t1 for _, _, t1 in tl)
    print(f"graph timeline: {end * 1e3:.1f} us")
    for name, t0, t1 in sorted(tl, key=lambda x: x[1]):
        print(f"  {t0 * 1e3:8.1f} {t1 * 1e3:8.1f} {1e3 * (t1 - t0):7.1f}  {name}")
