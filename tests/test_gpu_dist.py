"""Multi-rank path on the DEVICE (world 2, both ranks sharing cuda:0, gloo):
the per-rank CUDA pipeline on its stalled-PC shard (LeoConfig.consumer_lo/hi,
samples partitioned by owner of pc) plus the one all-reduce of the per-line
vectors reproduces the single-GPU result: blame entries concatenated in rank
order are bit-identical, the reduced line vectors equal the unsharded ones.
Then bench.py itself under torchrun --nproc-per-node 2 (LEO_BENCH_SHARE_GPU=1)
for the kernel-sharded C4 batch and the stalled-PC-sharded C5 kernel."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
SCALE = 0.02


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch.distributed as dist
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_20032_b200 import abi, device, synth
        from paper_2604_20032_b200 import dist as D
        dev = torch.device("cuda:0")
        wl = synth.config_workload("c5", scale=SCALE)
        (lo, hi), pc, cat = D.shard_workload(wl, rank, world)
        ks = wl.kernel
        dk = device.DeviceKernel(ks, dev)
        dp = device.DeviceProfile(wl.profile, ks.n_instr, dev)
        ds = device.DeviceSamples(pc, cat, wl.lut, dev)
        an = device.Analyzer(dk, dev, do_slice=False)
        an.run(dp, abi.make_config(dialect=ks.dialect, consumer_range=(lo, hi)), ds)
        r = an.result()
        lb, ls = an.line_blame.cpu(), an.line_stall.cpu()
        D.allreduce_lines(lb, ls)                   # the one collective
        q.put((rank, r["status"], r["e_stalled"].tolist(), r["e_blame"].tolist(),
               r["e_cause"].tolist(), lb.numpy().tolist(), ls.numpy().tolist()))
    finally:
        dist.destroy_process_group()


def test_device_stalled_pc_shards_world2_gloo():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    from paper_2604_20032_b200 import abi, device, synth
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=900) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    wl = synth.config_workload("c5", scale=SCALE)
    full = device.analyze_soa(wl.kernel, wl.profile, abi.make_config(dialect="nvidia"),
                              samples=(wl.pc, wl.cat, wl.lut), device=torch.device("cuda:0"))
    assert all(r[1] == 0 for r in res)
    assert [s for r in res for s in r[2]] == full["e_stalled"].tolist()
    assert [b for r in res for b in r[3]] == full["e_blame"].tolist()
    assert [c for r in res for c in r[4]] == full["e_cause"].tolist()
    assert res[0][5] == res[1][5] and res[0][6] == res[1][6]
    assert np.allclose(res[0][5], full["line_blame"], rtol=1e-12, atol=1e-9)
    assert np.allclose(res[0][6], full["line_stall"], rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("config,extra", [("c5", ["--scale", "0.05"]),
                                          ("c4", ["--c4-kernels", "12", "--scale", "0.25"])])
def test_bench_world2_shared_gpu(config, extra):
    """bench.py's N>1 path (torchrun, one rank per GPU, max-over-ranks timing,
    the all-reduce) run with both ranks on cuda:0."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, LEO_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--config", config, "--no-cpu", *extra]
    r = subprocess.run(cmd, cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
