#!/usr/bin/env python
"""PCIe bounds of the e2e step: 41 MB H2D (U, dU_prev) and 41 MB D2H (U', dU)
per step from pinned host memory, alone and concurrently on two streams."""
import time
import torch

n = 640000 * 4 * 2  # doubles: U + dU
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
B = n * 8


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


a, b, c = timed(h2d), timed(d2h), timed(both)
print(f"H2D {B / a / 1e9:.1f} GB/s ({a * 1e3:.3f} ms), D2H {B / b / 1e9:.1f} GB/s ({b * 1e3:.3f} ms), "
      f"both {c * 1e3:.3f} ms per step -> e2e bound {640000 / c / 1e6:.0f} Mpoint-it/s")
