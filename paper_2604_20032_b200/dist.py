"""Multi-GPU sharding of the hot path (one process per GPU, torch.distributed).

Two partitions, both with no data-path collective:

  * by kernel (C4, and the default bench: one kernel per rank) — kernels are
    independent; LPT assignment by estimated work;
  * by stalled-PC set (C5) — rank r owns the contiguous consumer range
    [lo_r, hi_r) balanced by use-unit count (a proxy for candidate edges).
    The instruction SoA, CFG and profile metadata are replicated; raw samples
    are pre-partitioned on the host by owner of `pc`; the device pipeline runs
    with LeoConfig.consumer_lo/hi so sync tracing, pruning, blame and the
    per-line stall rollup touch owned consumers only (raw/guard edges stay
    replicated: the indirect-addressing BFS of self-blame walks the unpruned
    RAW graph across shard boundaries, analysis.py:390-411).

The only exchange is one all-reduce (sum, f64) of the per-source-line blame
and stall vectors — NCCL over NVLink on GPUs, gloo in the CPU tests.
Per-instruction blame entries stay on their owner rank; concatenated in rank
order they equal the single-GPU entry list.
"""

from __future__ import annotations

import numpy as np


def consumer_ranges(ks, world: int) -> list[tuple[int, int]]:
    """Contiguous consumer ranges balanced by use-unit count (+1 per instruction)."""
    n = ks.n_instr
    op = np.asarray(ks.opnd, dtype=np.uint32)
    span = ((op >> 16) & 0xFF).astype(np.int64)
    use = ((op >> 27) & 3) != 2
    per_op = np.where(use, span, 0)
    owner = np.repeat(np.arange(n), np.diff(ks.opnd_ptr))
    w = np.bincount(owner, weights=per_op, minlength=n) + 1.0
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, cum[-1] * r / world)))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.asarray(cuts))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def partition_samples(pc: np.ndarray, ranges) -> list[np.ndarray]:
    """Index arrays of the raw samples each rank owns (owner of pc)."""
    bounds = np.asarray([lo for lo, _ in ranges[1:]], dtype=np.int64)
    owner = np.searchsorted(bounds, np.asarray(pc, dtype=np.int64), side="right")
    order = np.argsort(owner, kind="stable")
    counts = np.bincount(owner, minlength=len(ranges))
    splits = np.split(order, np.cumsum(counts)[:-1])
    return splits


def lpt_assign(costs, world: int) -> list[list[int]]:
    """Longest-processing-time-first assignment of independent kernels."""
    loads = [0.0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for k in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        r = min(range(world), key=lambda x: (loads[x], x))
        out[r].append(k)
        loads[r] += float(costs[k])
    for lst in out:
        lst.sort()
    return out


_EDGE_DENSITY = {"nvidia": 2.8, "amd": 2.6, "intel": 3.0}


def kernel_cost(dialect: str, n_instr: int) -> float:
    """Work estimate for LPT: instructions x expected candidate-edge density."""
    return n_instr * _EDGE_DENSITY.get(dialect, 3.0)


def allreduce_lines(line_blame, line_stall, group=None):
    """The single collective of the hot path: sum the per-line vectors."""
    import torch.distributed as dist
    dist.all_reduce(line_blame, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(line_stall, op=dist.ReduceOp.SUM, group=group)


def shard_workload(wl, rank: int, world: int):
    """Stalled-PC shard of one workload: (consumer range, pc, cat) for `rank`."""
    ranges = consumer_ranges(wl.kernel, world)
    idx = partition_samples(wl.pc, ranges)[rank]
    return ranges[rank], wl.pc[idx], wl.cat[idx]
