"""Host probe on the GPU box: cores, memory, NUMA placement of the GPU, and
the reference's setup / per-iteration cost on the config-4 / config-5 clouds
(decides what bench.py's reference arm and the config-4/5 parity tests can
afford). Usage: python scripts/probe_box.py [nw nr] ..."""
import os
import resource
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)


print(sh("nproc; free -g; lscpu | egrep 'Model name|Socket|Core|Thread|NUMA'; nvidia-smi topo -m; "
         "cat /sys/bus/pci/devices/$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | "
         "tr 'A-Z' 'a-z' | sed 's/^00000000/0000/')/numa_node"), flush=True)
import refpy  # noqa: E402

refpy.Reference.num_threads(os.cpu_count())
specs = [(int(sys.argv[i]), int(sys.argv[i + 1])) for i in range(1, len(sys.argv) - 1, 2)] or [(5120, 1920)]
for nw, nr in specs:
    t0 = time.perf_counter()
    ref = refpy.Reference.generate("0012", nw, nr, 20.0)
    t1 = time.perf_counter()
    print(f"ref generate {nw}x{nr}: n={ref.n} {t1 - t0:.1f}s maxrss {resource.getrusage(resource.RUSAGE_SELF).ru_maxrss/1e6:.1f} GB", flush=True)
    r = ref.run(variant="manish_ad", n_iterations=3, mach=0.63, aoa_deg=2.0, cfl=0.2)
    print(f"  run 3 its: seconds {list(r.seconds)} loop {r.loop_seconds:.1f}s wall {time.perf_counter()-t1:.1f}s "
          f"maxrss {resource.getrusage(resource.RUSAGE_SELF).ru_maxrss/1e6:.1f} GB", flush=True)
    del ref
import paper_2406_07441_b200 as kf  # noqa: E402
for nw, nr in specs:
    t0 = time.perf_counter()
    c = kf.generate_naca_ogrid("0012", nw, nr, 20.0)
    t1 = time.perf_counter()
    s = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2,
                                     n_iterations=3))
    t2 = time.perf_counter()
    h = s.run(want_state=False)
    print(f"ours {nw}x{nr}: generate {t1-t0:.1f}s solver {t2-t1:.1f}s run {time.perf_counter()-t2:.1f}s "
          f"its {len(h.iters)} maxrss {resource.getrusage(resource.RUSAGE_SELF).ru_maxrss/1e6:.1f} GB", flush=True)
    del s, c
