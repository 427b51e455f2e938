"""Per-iteration device time (globaltimer records of graph-launched
iterations) of the per-colour sweeps vs the dataflow sweeps (KF_SWEEP_DF) on
small clouds: BASELINE config 1 (the time-to-drop case) and larger NACA
O-grids up to config 2's size. Prints one line per (cloud, KF_SWEEP_DF)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2406_07441_b200 as kf  # noqa: E402

kf.Solver(kf.generate_naca_ogrid("0012", 48, 12, 12.0), kf.SolverConfig(n_iterations=2)).run()
for nw, nr in ((320, 120), (480, 160), (640, 320), (1600, 400)):
    c = kf.generate_naca_ogrid("0012", nw, nr, 20.0)
    res = {}
    for rep in range(2):
        for df in ("0", "1"):
            os.environ["KF_SWEEP_DF"] = df
            s = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0,
                                             cfl=0.2, n_iterations=150))
            os.environ.pop("KF_SWEEP_DF")
            s.run(want_state=False)
            h = s.run(want_state=False)
            sec = [r.seconds for r in h.iters[min(10, len(h.iters) - 1):]]
            res.setdefault(df, []).append(1e6 * float(np.median(sec)))
            del s
    for df, v in res.items():
        print(f"points {nw * nr:8d} KF_SWEEP_DF={df} median us/iteration " + " ".join(f"{x:.1f}" for x in v),
              flush=True)
