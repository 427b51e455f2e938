import time, os, sys
sys.path.insert(0, '/root/repo' if os.path.exists('/root/repo') else '.')
sys.path.insert(0, 'oracle')
os.environ["KF_TIME_INGEST"] = "1"
import paper_2406_07441_b200 as kf
def dropin(tag):
    t0 = time.perf_counter()
    c = kf.generate_naca_ogrid("0012", 320, 120, 20.0)
    t1 = time.perf_counter()
    s = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2, n_iterations=1000))
    t2 = time.perf_counter()
    h = s.run(want_state=True)
    t3 = time.perf_counter()
    print(tag, f"generate {t1-t0:.3f} solver {t2-t1:.3f} run {t3-t2:.3f}", flush=True)
dropin("fresh")
dropin("second")
import refpy
refpy.Reference.num_threads(16)
r = refpy.Reference.generate("0012", 320, 120, 20.0).run(variant="manish_ad", n_iterations=50, mach=0.63, aoa_deg=2.0, cfl=0.2)
dropin("after reference")
