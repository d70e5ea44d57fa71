"""Drive the fused pipeline for ncu: W eager warm-up steps, then K eager steps
(L2 flushed before each), one config.  Used as the <cmd> of the ncu launch
list / --set full captures committed under profiles/.

    python tools/profile_step.py [c2|c3|c5] [--steps K] [--warmup W] [--scale s]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2604_20032_b200 import abi, device, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c2")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--c4-kernels", type=int, default=300)
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--timeline", action="store_true")
ap.add_argument("--graph-timeline", action="store_true")
ap.add_argument("--phases", action="store_true")
ap.add_argument("--debug-guard", action="store_true")
args = ap.parse_args()

dev = torch.device("cuda:0")
if args.config == "c4":
    # the bench's C4 batch pipelines (one concatenated batch per dialect) over
    # the first --c4-kernels kernels of the 2,000
    from paper_2604_20032_b200 import batch as BT
    lines = synth.LineTable(4096, seed=999)
    groups = {}
    for kk in range(args.c4_kernels):
        w = synth.c4_kernel(kk, lines)
        groups.setdefault(BT.group_key(w), []).append(w)
    wls = [BT.concat(groups[key]) for key in sorted(groups)]
else:
    wls = [synth.config_workload(args.config, scale=args.scale)]
items = []
for wl in wls:
    dk = device.DeviceKernel(wl.kernel, dev)
    dp = device.DeviceProfile(wl.profile, wl.kernel.n_instr, dev)
    ds = device.DeviceSamples(wl.pc, wl.cat, wl.lut, dev)
    an = device.Analyzer(dk, dev, debug_flags=args.flags)
    cfg = abi.make_config(dialect=wl.kernel.dialect)
    an.run(dp, cfg, ds)                      # sizes buffers (grow + re-run on overflow)
    items.append((an, dp, cfg, ds))
wl = wls[0]
an, dp, cfg, ds = items[0]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(args.warmup):
    flush.zero_()
    for it in items:
        it[0].launch(*it[1:])
torch.cuda.synchronize()
for _ in range(args.steps):
    flush.zero_()
    for it in items:
        it[0].launch(*it[1:])
torch.cuda.synchronize()
for it in items:
    r = it[0].result()
    print(f"{args.config}: status={r['status']} edges={len(r['bprod'])} pruned={len(r['pprod'])} "
          f"blame={len(r['e_blame'])}")

if args.timeline:
    # eager step queued behind a GPU spin (so host launch overhead is hidden
    # and the branches run as they would in the graph), events per kernel
    tr = device.Tracer(capacity=4096, timeline=True)
    an.set_tracer(tr)
    for _ in range(3):
        tr.reset()
        flush.zero_()
        torch.cuda.synchronize()
        torch.cuda._sleep(20_000_000)
        an.launch(dp, cfg, ds)
        torch.cuda.synchronize()
    an.set_tracer(None)
    tl = tr.timeline()
    end = max(t1 for _, _, t1 in tl)
    print(f"timeline (eager step queued behind a spin, branches concurrent): {end * 1e3:.1f} us")
    for name, t0, t1 in sorted(tl, key=lambda x: x[1]):
        print(f"  {t0 * 1e3:8.1f} {t1 * 1e3:8.1f} {1e3 * (t1 - t0):7.1f}  {name}")

if args.graph_timeline:
    # the same, inside a CUDA graph replay (event-record nodes around kernels)
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

if args.phases:
    # per-CTA clock64 phase marks of the shared-memory tiers (LEO_DBG_PHASES)
    import numpy as np
    import ctypes as C
    from paper_2604_20032_b200._lib import lib
    an2 = device.Analyzer(dk, dev, debug_flags=args.flags | abi.DBG_PHASES)
    an2.run(dp, cfg, ds)
    flush.zero_()
    torch.cuda.synchronize()
    an2.launch(dp, cfg, ds)
    torch.cuda.synchronize()
    names = {0: ("reach_unit", ["staged", "near", "qlist", "queries"]),
             1: ("sync_wc_smem", ["staged", "events", "items", "ev_count", "ev_scan"]),
             2: ("prune_edges_smem", ["staged", "edges"])}
    for slot, (nm, ph) in names.items():
        buf = np.zeros((1024, 8), dtype=np.int64)
        lib().leo_debug_phases(slot, buf.ctypes.data_as(C.c_void_p), 1024)
        rows = buf[buf[:, len(ph)] > 0][:, 1:len(ph) + 1]
        if len(rows) == 0:
            print(f"{nm}: no marks")
            continue
        print(f"{nm}: {len(rows)} CTAs, cumulative clock64 at phase ends (median / max):")
        for i, p in enumerate(ph):
            print(f"   {p:10s} {int(np.median(rows[:, i])):9d} {int(rows[:, i].max()):9d}")
    it2 = np.zeros(16384, dtype=np.int64)
    lib().leo_debug_items.argtypes = [C.c_void_p, C.c_int32]
    lib().leo_debug_items(it2.ctypes.data_as(C.c_void_p), 16384)
    it = it2[:8192]
    rq = it2[8192:]
    rq = rq[rq > 0]
    if len(rq):
        cyc, nv = rq >> 24, rq & 0xFFFFFF
        o = np.argsort(-cyc)
        print(f"reach tier-0 queries: {len(rq)} (first 8192); cycles p50 {int(np.median(cyc))} p99 "
              f"{int(np.percentile(cyc, 99))} max {int(cyc.max())}; visits p50 {int(np.median(nv))} "
              f"p99 {int(np.percentile(nv, 99))} max {int(nv.max())}")
        print("  slowest (cycles, visits):", [(int(cyc[x]), int(nv[x])) for x in o[:12]])
        print("  cycles per visit (queries > 20 visits): p50",
              int(np.median(cyc[nv > 20] / nv[nv > 20])) if (nv > 20).any() else 0)
    wl_list = None
    order = np.argsort(-it)[:12]
    print("slowest waitcnt items (t*2+counter, cycles):", [(int(x), int(it[x])) for x in order])
    if (it > 0).any():
        print("item cycles: sum", int(it.sum()), "count>0", int((it > 0).sum()), "p50", int(np.median(it[it > 0])))

if args.debug_guard:
    import numpy as np
    import ctypes as C
    from paper_2604_20032_b200._lib import lib
    it = np.zeros(16, dtype=np.int64)
    lib().leo_debug_items.argtypes = [C.c_void_p, C.c_int32]
    lib().leo_debug_items(it.ctypes.data_as(C.c_void_p), 16)
    print("guard record:", it[:8].tolist())
