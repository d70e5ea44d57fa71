"""Host<->device copy bandwidth from pinned memory (the e2e path's transport).

    python tools/pcie_probe.py [--mb 400]

Times cudaMemcpyAsync H2D / D2H of one pinned buffer with CUDA events, plus
two concurrent H2D copies on two streams, so the e2e figures can be read
against what the link actually delivers on this box.
"""
import argparse

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--mb", type=int, default=400)
args = ap.parse_args()
n = args.mb << 20
dev = torch.device("cuda:0")
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n // 4, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device=dev)
d2 = torch.empty(n // 4, dtype=torch.uint8, device=dev)
h.fill_(1)


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


t = timed(lambda: d.copy_(h, non_blocking=True))
print(f"H2D {args.mb} MB pinned: {t * 1e3:.2f} ms  {n / t / 1e9:.1f} GB/s")
t = timed(lambda: h.copy_(d, non_blocking=True))
print(f"D2H {args.mb} MB pinned: {t * 1e3:.2f} ms  {n / t / 1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def two():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        d2.copy_(h2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t = timed(two)
print(f"H2D {args.mb}+{args.mb // 4} MB on two streams: {t * 1e3:.2f} ms  {(n + n // 4) / t / 1e9:.1f} GB/s")
hp = torch.empty(n, dtype=torch.uint8)           # pageable
t = timed(lambda: d.copy_(hp, non_blocking=True), reps=2)
print(f"H2D {args.mb} MB pageable: {t * 1e3:.2f} ms  {n / t / 1e9:.1f} GB/s")
