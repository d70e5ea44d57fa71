"""Device time of one pipeline step under CUDA graph replay (no trace events,
L2 flushed before each step), for A/B of library knobs.  Each variant runs in
its own process (the knobs are read once per process), interleaved R times.

    python tools/step_ab.py c5 "X=0" "LEO_T1=1" ... [--reps R] [--steps K]
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch
    from paper_2604_20032_b200 import abi, device, synth
    cfgname, steps = sys.argv[2], int(sys.argv[3])
    dev = torch.device("cuda:0")
    if cfgname.startswith("c4"):           # c4:K = the bench's batch pipelines over K kernels
        from paper_2604_20032_b200 import batch as BT
        K = int(cfgname.split(":")[1]) if ":" in cfgname else 300
        lines = synth.LineTable(4096, seed=999)
        groups = {}
        for kk in range(K):
            w = synth.c4_kernel(kk, lines)
            groups.setdefault(BT.group_key(w), []).append(w)
        wls = [BT.concat(groups[key]) for key in sorted(groups)]
    else:
        wls = [synth.config_workload(cfgname)]
    ans = []
    for wl in wls:
        dk = device.DeviceKernel(wl.kernel, dev)
        dp = device.DeviceProfile(wl.profile, wl.kernel.n_instr, dev)
        ds = device.DeviceSamples(wl.pc, wl.cat, wl.lut, dev)
        an = device.Analyzer(dk, dev)
        cfg = abi.make_config(dialect=wl.kernel.dialect)
        an.run(dp, cfg, ds)
        an.capture(dp, cfg, ds)
        ans.append((an, dk, dp, ds))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for s in range(steps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for x in ans:
            x[0].replay()
        b.record()
        torch.cuda.synchronize()
        if s >= 3:
            ts.append(a.elapsed_time(b))
    print(f"{np.median(ts) * 1e3:.1f} {np.min(ts) * 1e3:.1f}")
    sys.exit(0)

args = [a for a in sys.argv[1:] if not a.startswith("--")]
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 2
steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 20
cfgname, variants = args[0], [a for a in args[1:] if not a.isdigit()] or ["X=0"]
res = {v: [] for v in variants}
for r in range(reps):
    for v in variants:
        env = dict(os.environ)
        for kv in v.split():
            k, _, val = kv.partition("=")
            env[k] = val
        out = subprocess.run([sys.executable, __file__, "--child", cfgname, str(steps)], env=env,
                             capture_output=True, text=True, timeout=600)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else "ERR " + out.stderr[-300:]
        res[v].append(line)
for v in variants:
    print(f"{cfgname} {v:40s} median/min us: {' | '.join(res[v])}")
