#!/usr/bin/env python
"""Per-kernel device time of one iteration on BASELINE config 1 (38,400
points), where the time to a residual drop is measured: eager per-launch
CUDA events (kf_profile_kernels) and the graph-launched iteration time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_07441_b200 as kf  # noqa: E402

c = kf.generate_naca_ogrid("0012", 320, 120, 20.0)
cfg = kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2, n_iterations=1000)
s = kf.Solver(c, cfg)
s.reset()
s.iterate_async(20)
s.sync_records()
prof = s.profile_kernels(reps=20)
agg = {}
for name, ms in prof:
    agg.setdefault(name, []).append(ms)
tot = sum(ms for _, ms in prof)
for name, v in agg.items():
    print(f"{name:16s} launches {len(v):2d}  us/launch {1e3 * sum(v) / len(v):7.2f}  total {1e3 * sum(v):7.2f}")
print(f"eager sum {1e3 * tot:.1f} us per iteration")
h = s.run(want_state=False)
h = s.run(want_state=False)
sec = [r.seconds for r in h.iters[5:150]]
print(f"graph: {1e6 * sum(sec) / len(sec):.1f} us per iteration (device globaltimer between records)")
