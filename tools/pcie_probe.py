"""PCIe ceiling of the e2e path: pinned host <-> device copy bandwidth, one direction at a time
and both at once on two streams (the e2e pipeline's regime).  python tools/pcie_probe.py [GB]"""
import sys
import time

import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
n = int(gb * 2**30 / 8)
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


t_h2d = timed(lambda: d1.copy_(h1, non_blocking=True))
t_d2h = timed(lambda: h2.copy_(d2, non_blocking=True))
t_both = timed(both)
B = 8.0 * n / 1e9
print(f"H2D {B / t_h2d:.1f} GB/s, D2H {B / t_d2h:.1f} GB/s, both at once {B / t_both:.1f} GB/s per direction "
      f"({2 * B / t_both:.1f} GB/s total)")
