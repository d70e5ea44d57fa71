"""Time api.Session.analyze() call by call (status, retries, phases)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2604_20032_b200 import abi, api, device, synth

wl = synth.config_workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
dev = torch.device("cuda:0")
sess = api.Session(wl.kernel, wl.profile, wl.n_samples, abi.make_config(dialect=wl.kernel.dialect), dev)
sess.stage(wl.kernel, wl.profile, wl.pc, wl.cat, wl.lut)
orig_run = sess.an.run
calls = {"run": 0}
def run(*a, **k):
    calls["run"] += 1
    return orig_run(*a, **k)
sess.an.run = run
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sess.analyze()
    t1 = time.perf_counter()
    c = sess.an.ctr.cpu().numpy()
    print(f"call {it}: {1e3*(t1-t0):.2f} ms status={int(np.uint32(c[device.C_STATUS]))} runs={calls['run']} caps={sess.an.caps}")
# phases of one call
torch.cuda.synchronize(); t0 = time.perf_counter()
for n in sess.H2D_FIELDS:
    sess.dk.t[n].view(-1).copy_(sess._host["k_" + n], non_blocking=True)
torch.cuda.synchronize(); t1 = time.perf_counter()
S = sess.ds.n
sess.pc[:S].copy_(sess._host["pc"], non_blocking=True); sess.cat[:S].copy_(sess._host["cat"], non_blocking=True)
torch.cuda.synchronize(); t2 = time.perf_counter()
sess.an.launch(sess.dp, sess.cfg, sess.ds); torch.cuda.synchronize(); t3 = time.perf_counter()
out = sess.an.line_blame.to("cpu"); torch.cuda.synchronize(); t4 = time.perf_counter()
print(f"kernel h2d {1e3*(t1-t0):.2f} ms, samples h2d {1e3*(t2-t1):.2f} ms, launch {1e3*(t3-t2):.2f} ms, d2h {1e3*(t4-t3):.2f} ms")
print("pinned:", sess._host["pc"].is_pinned())
