"""Pinned host<->device copy rates on this box (the e2e bound): H2D alone,
D2H alone, both at once on two streams.

    python tools/pcie_probe.py [MB]
"""
import sys
import time

import torch

mb = int(sys.argv[1]) if len(sys.argv) > 1 else 460
n = mb << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, k=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


th = timed(lambda: d1.copy_(h1, non_blocking=True))
td = timed(lambda: h2.copy_(d2, non_blocking=True))
tb = timed(both)
print(f"{mb} MB pinned: H2D {n / th / 1e9:.1f} GB/s  D2H {n / td / 1e9:.1f} GB/s  "
      f"both {2 * n / tb / 1e9:.1f} GB/s aggregate ({tb * 1e3:.2f} ms for {mb} MB each way)")
