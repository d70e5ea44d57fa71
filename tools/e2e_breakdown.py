"""Where an api.Session.analyze() call spends its time (C2 by default):
graph replay + sync (device work + H2D / D2H inside the graph) versus the
host-side remainder of the call.

    python tools/e2e_breakdown.py [c2|c3|c5] [--calls N]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_20032_b200 import abi, api, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c2")
ap.add_argument("--calls", type=int, default=50)
args = ap.parse_args()
wl = synth.config_workload(args.config)
dev = torch.device("cuda:0")
sess = api.Session(wl.kernel, wl.profile, wl.n_samples, abi.make_config(dialect=wl.kernel.dialect), dev)
sess.stage(wl.kernel, wl.profile, wl.pc, wl.cat, wl.lut)
for _ in range(5):
    sess.analyze()
st = torch.cuda.current_stream()
t_call, t_replay, t_dev = [], [], []
for _ in range(args.calls):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sess.analyze()
    t_call.append(time.perf_counter() - t0)
for _ in range(args.calls):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    sess.graph.replay()
    e1.record()
    st.synchronize()
    t_replay.append(time.perf_counter() - t0)
    t_dev.append(e0.elapsed_time(e1) / 1e3)
med = lambda x: 1e6 * float(np.median(x))
print(f"{args.config}: analyze() {med(t_call):.1f} us | graph replay+sync (host) {med(t_replay):.1f} us | "
      f"graph on device (events) {med(t_dev):.1f} us | host remainder {med(t_call) - med(t_replay):.1f} us | "
      f"launch+sync overhead {med(t_replay) - med(t_dev):.1f} us")
