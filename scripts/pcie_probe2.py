#!/usr/bin/env python
"""Concurrent H2D + D2H rate of the config-5 e2e step (2.57 GB each way) for
three kinds of pinned host buffer: torch pin_memory (cudaHostAlloc), and
mmap'd buffers with / without transparent huge pages registered with
cudaHostRegister. Several repetitions each, interleaved, to see the spread."""
import ctypes
import mmap
import sys
import time

import torch

n_pts = int(sys.argv[1]) if len(sys.argv) > 1 else 40140800
nbytes = n_pts * 32  # one (n, 4) f64 array
cud = ctypes.CDLL("libcudart.so.12") if False else None
rt = torch.cuda.cudart()


def mm_buf(huge):
    m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    if huge:
        m.madvise(mmap.MADV_HUGEPAGE)
    t = torch.frombuffer(m, dtype=torch.float64)
    t.fill_(1.0)  # touch
    r = rt.cudaHostRegister(t.data_ptr(), nbytes, 0)
    assert int(r) == 0, r
    return t, m


def make(kind):
    if kind == "pin":
        return [torch.empty(nbytes // 8, dtype=torch.float64).pin_memory() for _ in range(4)], None
    bufs = [mm_buf(kind == "thp") for _ in range(4)]
    return [b[0] for b in bufs], [b[1] for b in bufs]


dev = [torch.empty(nbytes // 8, dtype=torch.float64, device="cuda") for _ in range(4)]
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def run(h, mode, rounds=4):
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    s_in.wait_event(e0)
    s_out.wait_event(e0)
    for _ in range(rounds):
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s_in):
                dev[0].copy_(h[0], non_blocking=True)
                dev[1].copy_(h[1], non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s_out):
                h[2].copy_(dev[2], non_blocking=True)
                h[3].copy_(dev[3], non_blocking=True)
    e1.record(s_in)
    e2.record(s_out)
    torch.cuda.synchronize()
    return max(e0.elapsed_time(e1), e0.elapsed_time(e2)) / rounds


kinds = ["pin", "mmap4k", "thp"]
H = {}
for k in kinds:
    t = time.perf_counter()
    H[k] = make(k)
    print(f"{k}: alloc+pin {time.perf_counter() - t:.2f} s", flush=True)
for rep in range(3):
    for k in kinds:
        h = H[k][0]
        a, b, c = run(h, "h2d"), run(h, "d2h"), run(h, "both")
        print(f"rep {rep} {k:7s} h2d {2 * nbytes / a / 1e6:5.1f} GB/s  d2h {2 * nbytes / b / 1e6:5.1f} GB/s  "
              f"both {c:6.1f} ms/step ({2 * nbytes / c / 1e6:5.1f} GB/s each way)", flush=True)
