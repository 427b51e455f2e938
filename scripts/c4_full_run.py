"""Evidence (GPU box): BASELINE config 4 (NACA 0012 5120x1920, 9,830,400
points, M 0.63, AoA 2, manish_ad, CFL 0.2) run to its end on the B200 and by
the unmodified reference on the host cores (~3.2 s per reference iteration):
whole residual / CL / CD histories, first-order counts and the abort record.
Writes one JSON object (argv[1]). C4_CLOUD=nw:nr and C4_ITERS select another
cloud / iteration count (config 5: 10240:3920, 30 iterations -- the bench's
timed window)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2406_07441_b200 as kf  # noqa: E402
import refpy  # noqa: E402

N_IT = int(os.environ.get("C4_ITERS", "140"))
NW, NR = (int(v) for v in os.environ.get("C4_CLOUD", "5120:1920").split(":"))
cfg = kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2, n_iterations=N_IT)
t0 = time.perf_counter()
c = kf.generate_naca_ogrid("0012", NW, NR, 20.0)
g = kf.Solver(c, cfg).run()
t1 = time.perf_counter()
refpy.Reference.num_threads(os.cpu_count() or 1)
r = refpy.Reference.generate("0012", NW, NR, 20.0).run(variant="manish_ad", n_iterations=N_IT, mach=0.63,
                                                            aoa_deg=2.0, cfl=0.2)
t2 = time.perf_counter()
n = min(len(g.iters), len(r.residual))
rel = float(np.max(np.abs(g.residual[:n] - r.residual[:n]) / np.abs(r.residual[:n]))) if n else None
out = {"config": f"naca0012:{NW}:{NR}:20 M0.63 AoA2 manish_ad CFL0.2", "points": c.n(), "n_iterations": N_IT,
       "gpu_iterations": len(g.iters), "ref_iterations": int(len(r.residual)),
       "gpu_abort": g.abort_reason, "ref_abort": r.abort_reason,
       "residual_rel_max": rel,
       "cl_abs_max": float(np.max(np.abs(g.cl[:n] - r.cl[:n]))) if n else None,
       "cd_abs_max": float(np.max(np.abs(g.cd[:n] - r.cd[:n]))) if n else None,
       "first_order_equal": bool(np.array_equal(g.first_order[:n], r.first_order[:n])),
       "gpu_loop_seconds": g.loop_seconds, "ref_loop_seconds": r.loop_seconds,
       "gpu_wall_with_setup": t1 - t0, "ref_wall_with_setup": t2 - t1,
       "decades_reached": float(np.log10(r.residual[0] / np.min(r.residual))) if n else None,
       # per-iteration relative residual error (where a chaotic approach to
       # the abort amplifies the few-ulp differences)
       "residual_rel_per_iteration": [float(v) for v in np.abs(g.residual[:n] - r.residual[:n]) / np.abs(r.residual[:n])],
       "gpu_residual": [float(v) for v in g.residual], "ref_residual": [float(v) for v in r.residual]}
print(json.dumps(out))
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)
