"""Work routed to each search tier (LEO_DBG_PHASES counters) for a config.

    python tools/tier_counts.py c2|c3|c5 [--scale s] | c4 <n_kernels>
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_20032_b200 import abi, batch, device, synth  # noqa: E402
from paper_2604_20032_b200._lib import lib  # noqa: E402

dev = torch.device("cuda:0")
if sys.argv[1] == "c4":
    lines = synth.LineTable(256, seed=999)
    groups = {}
    for k in range(int(sys.argv[2])):
        wl = synth.c4_kernel(k, lines)
        groups.setdefault(batch.group_key(wl), []).append(wl)
    items = [(key, batch.concat(g)) for key, g in sorted(groups.items())]
else:
    scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    wl = synth.config_workload(sys.argv[1], scale=scale)
    items = [((wl.kernel.dialect,), wl)]
L = lib()
L.leo_debug_tiers.argtypes = [C.c_void_p]
for key, wl in items:
    dk = device.DeviceKernel(wl.kernel, dev)
    dp = device.DeviceProfile(wl.profile, wl.kernel.n_instr, dev)
    ds = device.DeviceSamples(wl.pc, wl.cat, wl.lut, dev)
    an = device.Analyzer(dk, dev, debug_flags=abi.DBG_PHASES)
    an.run(dp, abi.make_config(dialect=wl.kernel.dialect), ds)
    c = np.zeros(16, dtype=np.int32)
    L.leo_debug_tiers(c.ctypes.data_as(C.c_void_p))
    print(key, f"N={wl.kernel.n_instr} B={wl.kernel.n_blocks}", "queries", c[0], "reach_t2", c[2], "reach_t3", c[7],
          "waits", c[8], "wc_warp", c[10], "sync_exact", c[4], "sync_keys", c[3])
