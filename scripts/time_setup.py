"""Host setup time of a large cloud: ingestion (generate + split + LS +
colouring) and the device packing (layout, tiles, weight streams, upload)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["KF_TIME_INGEST"] = "1"
import paper_2406_07441_b200 as kf
nw, nr = (int(v) for v in sys.argv[1].split(":"))
t0 = time.time()
c = kf.generate_naca_ogrid("0012", nw, nr, 20.0)
t1 = time.time()
s = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, n_iterations=10))
t2 = time.time()
import resource
ru = resource.getrusage(resource.RUSAGE_SELF)
print(f"points {c.n()} ingest {t1 - t0:.2f} s solver {t2 - t1:.2f} s (process user {ru.ru_utime:.1f} s, "
      f"sys {ru.ru_stime:.1f} s, max rss {ru.ru_maxrss / 1e6:.1f} GB)", flush=True)
