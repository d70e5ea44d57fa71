"""Multi-process sharding logic on CPU (gloo, world_size 2).

The per-shard analysis here is the oracle restricted to the shard's owned
consumers (test infrastructure); the GPU shard path is checked in
tests/test_gpu_parity.py::test_device_consumer_shards_recombine.  What these
tests pin: the consumer-range and sample partitions, LPT kernel assignment,
and that the single all-reduce of per-line vectors reproduces the
single-process totals.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_20032_b200 import dist as D
from paper_2604_20032_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_consumer_ranges_partition_everything():
    wl = synth.config_workload("c5", scale=0.01)
    for world in (1, 2, 3, 8):
        r = D.consumer_ranges(wl.kernel, world)
        assert r[0][0] == 0 and r[-1][1] == wl.kernel.n_instr
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        parts = D.partition_samples(wl.pc, r)
        allidx = np.sort(np.concatenate(parts))
        assert np.array_equal(allidx, np.arange(wl.pc.shape[0]))
        for (lo, hi), idx in zip(r, parts):
            assert np.all((wl.pc[idx] >= lo) & (wl.pc[idx] < hi))


def test_lpt_assigns_each_kernel_once_and_balances():
    costs = [D.kernel_cost(d, n) for d, n in
             zip(["nvidia", "amd", "intel"] * 10, np.random.default_rng(0).integers(100, 5000, 30))]
    for world in (1, 2, 4, 8):
        a = D.lpt_assign(costs, world)
        flat = sorted(k for lst in a for k in lst)
        assert flat == list(range(len(costs)))
        loads = [sum(costs[k] for k in lst) for lst in a]
        assert max(loads) - min(loads) <= max(costs) + 1e-9


def _shard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        wl = synth.config_workload("c5", scale=0.005)
        ks = wl.kernel
        (lo, hi), pc, cat = D.shard_workload(wl, rank, world)
        # the shard bins only its own samples
        lat, cls = oracle.bin_samples(pc, cat, wl.lut, ks.n_instr)
        assert np.all(lat[:lo] == 0) and np.all(lat[hi:] == 0)
        p = wl.profile
        prof = type(p)(period=p.period, lat=lat, cls_cnt=cls, exec_cnt=p.exec_cnt,
                       total=p.total, eff=p.eff, sampled=p.sampled)
        r = oracle.run(ks, prof)
        own = (r.e_stalled >= lo) & (r.e_stalled < hi)
        at = np.where(r.e_edge[own] < 0, r.e_stalled[own], r.p_prod[np.maximum(r.e_edge[own], 0)])
        L = len(ks.lines)
        lb = np.zeros(L)
        np.add.at(lb, ks.line_id[at], r.e_blame[own])
        ls = np.zeros(L)
        j = np.arange(lo, hi)
        np.add.at(ls, ks.line_id[j], lat[lo:hi].astype(np.float64) * p.period)
        tb, tsl = torch.from_numpy(lb), torch.from_numpy(ls)
        D.allreduce_lines(tb, tsl)
        q.put((rank, r.e_stalled[own].tolist(), r.e_blame[own].tolist(), tb.numpy().tolist(),
               tsl.numpy().tolist()))
    finally:
        dist.destroy_process_group()


def test_stalled_pc_sharding_gloo_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import oracle
    wl = synth.config_workload("c5", scale=0.005)
    full = oracle.run(wl.kernel, synth.bin_host(wl))
    stalled = [s for r in res for s in r[1]]
    blame = [b for r in res for b in r[2]]
    # per-instruction blame is exact and, concatenated in rank order, equals the unsharded list
    assert stalled == full.e_stalled.tolist()
    assert blame == full.e_blame.tolist()
    # the all-reduced line vectors are identical on both ranks and match the oracle
    assert res[0][3] == res[1][3] and res[0][4] == res[1][4]
    assert np.allclose(res[0][3], full.line_blame, rtol=1e-12, atol=1e-9)
    assert np.allclose(res[0][4], full.line_stall, rtol=1e-12, atol=1e-9)
