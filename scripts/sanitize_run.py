"""A few iterations of every transport under compute-sanitizer (memcheck/racecheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_07441_b200 as kf
c = kf.generate_naca_ogrid("0012", 64, 16, 12.0)
for env in ({}, {"KF_RES_SPLIT_MAX": "0"}, {"KF_FLUX_KERNEL": "m3"}, {"KF_GATHER": "ell"}):
    # two-thread (small-cloud) and one-thread flux kernels, the exact variant,
    # the global-gather kernels
    for k in ("KF_RES_SPLIT_MAX", "KF_FLUX_KERNEL", "KF_GATHER"):
        os.environ.pop(k, None)
    os.environ.update(env)
    for variant in ("manish_ad", "anandh", "explicit"):
        cfg = kf.SolverConfig(variant=kf.SolverVariant.parse(variant), mach_inf=0.63, aoa_deg=2.0,
                              cfl=0.05 if variant == "explicit" else 0.2, n_iterations=6)
        for parts in (1, 3):
            r = kf.Solver(c, cfg, n_parts=parts).run()
            print(env, variant, parts, len(r.iters), r.abort_reason, flush=True)
for k in ("KF_RES_SPLIT_MAX", "KF_FLUX_KERNEL", "KF_GATHER"):
    os.environ.pop(k, None)
s = kf.Solver.for_rank(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, n_iterations=4), 1, 0, kf.nccl_unique_id())
print("nccl", len(s.run().iters))
s = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, n_iterations=8))
s.reset(); s.iterate_async(2); U, dU = s.get_state(with_dU=True)
outs = [np.zeros_like(U) for _ in range(3)]
s.step_host_batch([U] * 3, [dU] * 3, outs, [np.zeros_like(U) for _ in range(3)])
s.bench_mode(True); s.iterate_async(2); print("bench", s.sync_records()[1].code)
# round 2: device colouring (Jones-Plassmann + iterated greedy) and the
# wall-first levels, the overlapped exchanges (in-process, forced on), and a
# cloud wide enough for many tiles (device-built weight streams)
c2 = kf.generate_naca_ogrid("0012", 160, 41, 20.0)
kf.color_points_device(c2, "ldf")
kf.order_wall_first(c2)
cfg = kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, n_iterations=4)
print("ordering variant", len(kf.Solver(c2, cfg).run().iters))
os.environ["KF_OVERLAP"] = "1"
for variant in ("manish_ad", "anandh"):
    cfg = kf.SolverConfig(variant=kf.SolverVariant.parse(variant), mach_inf=0.63, aoa_deg=2.0, n_iterations=4)
    print("overlap", variant, len(kf.Solver(kf.generate_naca_ogrid("0012", 160, 41, 20.0), cfg, n_parts=3).run().iters))
os.environ.pop("KF_OVERLAP")
# dataflow sweeps (KF_SWEEP_DF=1: ticketed blocks, per-slice release flags)
os.environ["KF_SWEEP_DF"] = "1"
for variant in ("manish_ad", "anandh"):
    cfg = kf.SolverConfig(variant=kf.SolverVariant.parse(variant), mach_inf=0.63, aoa_deg=2.0, n_iterations=4)
    print("dataflow", variant, len(kf.Solver(kf.generate_naca_ogrid("0012", 160, 41, 20.0), cfg).run().iters))
os.environ.pop("KF_SWEEP_DF")
print("done")
