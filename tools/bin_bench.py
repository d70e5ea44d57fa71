"""Stage-0 binning alone (leo_bin_samples) on a config's raw sample stream:
device time per call (CUDA events, L2 flushed before each), effective GB/s
over the 5 bytes per sample, checked against a host bincount.  Table geometry
A/B: LEO_BIN_SLOTS / LEO_BIN_PROBE.

    python tools/bin_bench.py [c5|c3|c2] [--iters K]
"""
import argparse
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_20032_b200 import device, synth  # noqa: E402
from paper_2604_20032_b200._lib import lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c5")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--variants", default="")
args = ap.parse_args()
dev = torch.device("cuda:0")
wl = synth.config_workload(args.config)
N, S = wl.kernel.n_instr, wl.n_samples
ds = device.DeviceSamples(wl.pc, wl.cat, wl.lut, dev)
cls = torch.zeros(N * 8, dtype=torch.int32, device=dev)
lat = torch.zeros(N, dtype=torch.int32, device=dev)
status = torch.zeros(1, dtype=torch.int32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
L = lib()
want = np.bincount(wl.pc.astype(np.int64) * 8 + wl.lut[wl.cat].astype(np.int64), minlength=N * 8)
st = torch.cuda.current_stream().cuda_stream


def call():
    rc = L.leo_bin_samples(C.byref(ds.struct), N, C.c_void_p(lat.data_ptr()), C.c_void_p(cls.data_ptr()),
                           C.c_void_p(status.data_ptr()), C.c_void_p(st))
    assert rc == 0


call()
torch.cuda.synchronize()
assert np.array_equal(cls.cpu().numpy(), want), "binning mismatch"
ts = []
for _ in range(args.iters):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    call()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = float(np.median(ts))
print(f"{args.config} S={S} slots={os.environ.get('LEO_BIN_SLOTS', 'default')} "
      f"probe={os.environ.get('LEO_BIN_PROBE', 'default')}: {ms * 1e3:.1f} us "
      f"({5 * S / ms / 1e6:.0f} GB/s of samples, memset+hash+finalize) ok")
