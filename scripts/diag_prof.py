import sys, time
sys.path.insert(0, '/root/repo')
import paper_2406_07441_b200 as kf
c = kf.generate_naca_ogrid("0012", 1280, 500, 20.0)
cfg = kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.85, aoa_deg=1.0, cfl=0.2, n_iterations=64)
s = kf.Solver(c, cfg)
s.reset(); s.iterate_async(5); s.sync_records(); s.bench_mode(True)
for r in (1, 5, 20, 20):
    prof = s.profile_kernels(reps=r)
    print(r, [(n, round(t, 4)) for n, t in prof])
