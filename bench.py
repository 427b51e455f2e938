#!/usr/bin/env python
"""Benchmark of the B200 implicit-LSKUM hot path (one JSON line on rank 0).

Workload (BASELINE.json configs[1]): NACA 0012 O-grid 1280x500 (640,000
points, radius 20), M 0.85, AoA 1 deg, modified LU-SGS with exact-AD JVPs
(manish_ad), CFL 0.2, 3 inner gradient passes, physical BCs. A *step* is one
fixed-point iteration (driver.cpp:218-276): q, 3 q-derivative passes, split-
flux residual, time step + S-term + diagonal, 4 forward and 3 backward colour
sweeps, update + BCs, residual norm and CL/CD.

The reference aborts this case during iteration 22, so a
long trajectory cannot be timed. Every timed step therefore re-runs iteration
6 from the resident iteration-5 state (kf_bench_mode: the restart copy of U
and dU_prev is inside the timed step).

  value : device-timed Mpoint-iter/s (CUDA events on the library stream,
          state resident in HBM), whole job over all ranks.
  e2e   : the same metric through the reference-facing C-ABI call
          kf_step_host with pinned HOST buffers: H2D(U, dU_prev) + iteration +
          D2H(U', dU, record) every step.

Multi-GPU (--gpus N under torchrun, one process per GPU): the domain-
decomposed solver. The cloud grows with N (n_wall = 1280 N,
so every GPU owns ~640,000 points: weak scaling), is cut into N angular
wedges, and every rank solves its wedge with ghost points refreshed by grouped
ncclSend/ncclRecv between dependent stages plus one ncclAllReduce of the
residual/forces/abort partials per iteration. `value` is all ranks' points
times steps over the max-over-ranks device time.

--parts P (single process) runs the same decomposition in-process on one GPU
(ghosts refreshed by device copies): the partitioning overhead on one B200.

--impl reference times the reference's own CPU solver (oracle/_ref, all host
threads) on the same case.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs (SURVEY.md §8(d) clouds); 2 is the bench workload,
# the others are reachable with --case for evidence runs
CASES = {
    2: dict(digits="0012", n_wall=1280, n_radial=500, radius=20.0, mach=0.85, aoa=1.0, cfl=0.2,
            variant="manish_ad"),
    3: dict(digits="0012", n_wall=2560, n_radial=960, radius=20.0, mach=1.2, aoa=0.0, cfl=0.2,
            variant="anandh_ad"),
    4: dict(digits="0012", n_wall=5120, n_radial=1920, radius=20.0, mach=0.63, aoa=2.0, cfl=0.2,
            variant="manish_ad"),
    5: dict(digits="0012", n_wall=10240, n_radial=3920, radius=20.0, mach=0.63, aoa=2.0, cfl=0.2,
            variant="manish_ad"),
}
CASE = dict(digits="0012", n_wall=1280, n_radial=500, radius=20.0, mach=0.85, aoa=1.0, cfl=0.2,
            variant="manish_ad")
METRIC = "Mpoint-iter/s (FP64 LU-SGS+AD) and time-to-residual-drop, NACA 0012 clouds"
UNIT = "Mpoint-iter/s"
WARM_ITERS = 5
# algorithmic bytes of the flux-residual kernel per point
# (q 32 + qx,qy 64 + xy 16 + ids 4*n_s + R 32, n_s = split entries with w != 0)
FLUX_BYTES_FIXED = 144.0
# whole iteration, n_inner = 3, Manish: 144 + 2x176 + 144 + 176 + 121 + 121 + 97
ITER_BYTES_FIXED = 1155.0


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region, through
    NVML (pynvml, ~1 ms per query, every 5 ms) so even a short timed region
    gets many samples; nvidia-smi as the fallback."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self.nv = None

    def _nvml(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.005)

    def _smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "sw_thermal_slowdown", "hw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + fields,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                r = [x.strip() for x in out.split(",")]
                self.sm.append(float(r[0]))
                self.mx.append(float(r[1]))
                for k, nm in enumerate(names):
                    if r[2 + k].lower() == "active":
                        self.reasons.add(nm)
            except Exception:
                pass
            self._stop.wait(0.05)

    def start(self):
        self._t = threading.Thread(target=self._nvml if self.nv else self._smi, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None,
                "sm_max_mhz": float(max(self.mx)) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self.nv else "nvidia-smi"}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_cpu(n_iters_total, threads, spec=CASE):
    """Time the reference solver (oracle/_ref, else the C restatement) on the
    case. Returns (per-iteration seconds excluding each run's iteration 1,
    N, kind). Runs restart from freestream before the reference's abort
    (iteration 22) so any number of iterations can be sampled."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refpy  # checker: only the cpu_baseline / reference arm may use it
    kind = "reference" if refpy.ref_available() else "port"
    if kind == "reference":
        refpy.Reference.num_threads(threads)
        ctx = refpy.Reference.generate(spec["digits"], spec["n_wall"], spec["n_radial"], spec["radius"])
    else:
        os.environ["OMP_NUM_THREADS"] = str(threads)
        import paper_2406_07441_b200 as kf
        c = kf.generate_naca_ogrid(spec["digits"], spec["n_wall"], spec["n_radial"], spec["radius"])
        nb = c.nbr
        ctx = refpy.Oracle(c.x, c.y, c.kind, c.normal_x, c.normal_y, nb.offsets, nb.ids)
    secs = []
    while len(secs) < n_iters_total:
        m = min(n_iters_total - len(secs) + 1, 20)
        t0 = time.perf_counter()
        r = ctx.run(variant=spec["variant"], n_iterations=m, mach=spec["mach"], aoa_deg=spec["aoa"],
                    cfl=spec["cfl"])
        wall = time.perf_counter() - t0
        s = list(r.seconds[1:]) if kind == "reference" else [wall / max(len(r.residual), 1)] * (len(r.residual) - 1)
        if not s:
            break
        secs.extend(s)
    return secs[:n_iters_total], ctx.n, kind


def time_to_drop(kf, decades=1.0, with_cpu=True):
    """Time to a fixed residual drop (north star; RunHistory::iterations_to_decades,
    driver.cpp:169-178) on BASELINE config 1 (NACA 0012 320x120, M 0.63, AoA 2,
    manish_ad, CFL 0.2): the reference reaches ~1 decade before its abort in
    iteration 423, so 10 decades is not reachable; the drop
    reported is `decades`. GPU: device seconds of the iterations up to the
    drop (per-iteration globaltimer records). CPU: the reference solver's own
    per-iteration seconds for the same iterations, all host threads."""
    c = kf.generate_naca_ogrid("0012", 320, 120, 20.0)
    cfg = kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2,
                          n_iterations=1000)
    s = kf.Solver(c, cfg)
    s.run(want_state=False)  # warm-up (graphs, caches)
    h = s.run(want_state=False)
    k = h.iterations_to_decades(decades)
    out = {"config": "naca0012:320:120:20 M0.63 AoA2 manish_ad CFL0.2", "decades": decades,
           "iterations": k, "recorded_iterations": len(h.iters), "abort": h.abort_reason}
    if k <= 0:
        return out
    out["gpu_seconds"] = float(sum(r.seconds for r in h.iters[:k]))
    if with_cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import refpy
        if refpy.ref_available():
            refpy.Reference.num_threads(cpu_cores())
            ref = refpy.Reference.generate("0012", 320, 120, 20.0)
            r = ref.run(variant="manish_ad", n_iterations=k, mach=0.63, aoa_deg=2.0, cfl=0.2)
            out["cpu_seconds"] = float(np.sum(r.seconds[:k]))
            out["cpu_kind"] = "reference"
            out["cpu_cores"] = cpu_cores()
            out["speedup"] = out["cpu_seconds"] / out["gpu_seconds"]
    return out


def shuffled(kf, c, seed=7):
    """The same cloud under a random point numbering (kf_cloud_from_arrays
    rebuilds split stencils, LS weights and the greedy colouring)."""
    n = c.n()
    # wall points keep their (surface-ordered) ids so compute_forces' loop
    # check holds; every other point gets a random id
    wall = np.flatnonzero(c.kind == 0)
    rest = np.setdiff1d(np.arange(n), wall)
    perm = np.concatenate([wall, np.random.default_rng(seed).permutation(rest)])  # new id -> old id
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    nb = c.nbr
    deg = np.diff(nb.offsets)[perm]
    off = np.zeros(n + 1, np.int32)
    np.cumsum(deg, out=off[1:])
    ids = np.concatenate([inv[nb.ids[nb.offsets[o]:nb.offsets[o + 1]]] for o in perm]).astype(np.int32)
    return kf.PointCloud.from_arrays(c.x[perm], c.y[perm], c.kind[perm].astype(np.int32), c.normal_x[perm],
                                     c.normal_y[perm], off, ids)


def case_for(world, points=None, case=2):
    """The bench workload at `world` GPUs: config 2 at N=1; the cloud grows
    with N in the wall direction (weak scaling, ~640,000 points per GPU)."""
    spec = dict(CASES[case])
    spec["n_wall"] = spec["n_wall"] * max(world, 1)
    if points:
        nw, nr = points.split(":")
        spec["n_wall"], spec["n_radial"] = int(nw), int(nr)
    return spec


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = cpu_cores()
    spec = case_for(world, args.points, args.case)
    secs, n, kind = reference_cpu(args.warmup + args.steps, threads, spec)
    timed = secs[args.warmup:args.warmup + args.steps] or secs
    total = float(np.sum(timed))
    value = n * len(timed) / total / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(timed), "warmup": args.warmup, "ms_per_step": 1e3 * total / len(timed),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated NACA 0012 O-grid, deterministic)",
        "config": {"workload": f"naca0012:{spec['n_wall']}:{spec['n_radial']}:20 M{spec['mach']} "
                               f"AoA{spec['aoa']:g} {spec['variant']} CFL{spec['cfl']}, one fixed-point iteration",
                   "points": n, "parallelism": "cpu-openmp"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{len(timed)} reference iterations of the same case (runs restarted "
                                   f"from freestream every <=19 iterations; iteration 1 of each run excluded)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true",
                    help="run a few steps for ncu (no JSON line)")
    ap.add_argument("--points", default=None, help="override cloud n_wall:n_radial")
    ap.add_argument("--parts", type=int, default=1, help="in-process partitions on one GPU")
    ap.add_argument("--variant", default=None,
                    choices=["explicit", "anandh", "anandh_ad", "manish", "manish_ad"],
                    help="override the case's solver variant (evidence runs)")
    ap.add_argument("--ordering", type=int, default=1, choices=[0, 1, 2],
                    help="in-colour point order: 0 natural, 1 Morton (default), 2 reverse Cuthill-McKee")
    ap.add_argument("--shuffle", action="store_true",
                    help="randomly renumber the cloud's points first (a loaded cloud with no locality: "
                         "the --ordering demonstration)")
    ap.add_argument("--case", type=int, default=2, choices=sorted(CASES),
                    help="BASELINE.json config whose cloud/case to time (default 2, the bench workload)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import paper_2406_07441_b200 as kf

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec = case_for(world, args.points, args.case)
    if args.variant:
        spec["variant"] = args.variant

    cloud = kf.generate_naca_ogrid(spec["digits"], spec["n_wall"], spec["n_radial"], spec["radius"])
    if args.shuffle:
        cloud = shuffled(kf, cloud)
    N = cloud.n()
    cfg = kf.SolverConfig(variant=kf.SolverVariant.parse(spec["variant"]), mach_inf=spec["mach"],
                          aoa_deg=spec["aoa"], cfl=spec["cfl"], n_iterations=64, device=local,
                          ordering=args.ordering)
    if world > 1:
        ids = [kf.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(ids, src=0)
        solver = kf.Solver.for_rank(cloud, cfg, world, rank, ids[0])
    else:
        solver = kf.Solver(cloud, cfg, n_parts=args.parts)
    solver.reset()
    solver.iterate_async(WARM_ITERS)
    recs, st = solver.sync_records()
    assert st.code == 0 and len(recs) == WARM_ITERS, st.reason
    # the resident iteration-5 state: every timed step (device and e2e) runs
    # iteration 6 from it
    U0, dU0 = solver.get_state(with_dU=True)
    solver.bench_mode(True)
    stream = torch.cuda.ExternalStream(solver.stream_ptr, device=torch.device("cuda", local))

    if args.profile_only:
        solver.iterate_async(args.warmup + args.steps)
        solver.sync_records()
        torch.cuda.synchronize()
        return 0

    # ---- device-timed steps
    solver.iterate_async(args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(stream)
    solver.iterate_async(args.steps)
    t1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = t0.elapsed_time(t1)
    recs, st = solver.sync_records()
    if st.code != 0:
        raise RuntimeError("benchmark iteration failed: " + st.reason.decode())
    ms_t = torch.tensor([ms], device="cuda")
    if world > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = N * args.steps / (ms_max * 1e-3) / 1e6  # N: points of the whole (all-rank) cloud
    launches = solver.launches_per_iteration * args.steps

    # ---- end to end through the C ABI with pinned host buffers
    Uh = torch.from_numpy(U0).pin_memory()
    dUh = torch.from_numpy(dU0).pin_memory()
    Uo = torch.empty_like(Uh).pin_memory()
    dUo = torch.empty_like(dUh).pin_memory()
    import ctypes as C
    from paper_2406_07441_b200 import _lib
    rec = _lib.IterRecord()
    h = solver._h

    def e2e_step():
        s = _lib.lib.kf_step_host(h, C.c_void_p(Uh.data_ptr()), C.c_void_p(dUh.data_ptr()),
                                  C.c_void_p(Uo.data_ptr()), C.c_void_p(dUo.data_ptr()), C.byref(rec))
        if s.code != 0:
            raise RuntimeError(s.reason.decode())

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    # synchronous form: one blocking C-ABI call per step
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    sync_ms = max(e0.elapsed_time(e1), 1e3 * wall)
    # pipelined form (kf_step_host_batch): the same steps, H2D of step k+1 and
    # D2H of step k-1 on the copy engines while step k computes
    Uos = [torch.empty_like(Uh).pin_memory() for _ in range(2)]
    dUos = [torch.empty_like(dUh).pin_memory() for _ in range(2)]
    recs_b = (_lib.IterRecord * args.steps)()

    def batch(m):
        P = C.c_void_p * m
        s = _lib.lib.kf_step_host_batch(h, m, P(*[Uh.data_ptr()] * m), P(*[dUh.data_ptr()] * m),
                                        P(*[Uos[k & 1].data_ptr() for k in range(m)]),
                                        P(*[dUos[k & 1].data_ptr() for k in range(m)]), recs_b)
        if s.code != 0:
            raise RuntimeError(s.reason.decode())

    batch(args.warmup)
    torch.cuda.synchronize()
    # host wall clock around the blocking batch call; the median of three
    # batches (the PCIe-bound step varies by several % from run to run)
    walls = []
    for _ in range(3):
        w0 = time.perf_counter()
        batch(args.steps)
        torch.cuda.synchronize()
        walls.append(1e3 * (time.perf_counter() - w0))
    e2e_ms = float(np.median(walls))
    et = torch.tensor([e2e_ms, sync_ms], device="cuda")
    if world > 1:
        torch.distributed.all_reduce(et, op=torch.distributed.ReduceOp.MAX)
    e2e_value = N * args.steps / (float(et[0].item()) * 1e-3) / 1e6
    e2e_sync_value = N * args.steps / (float(et[1].item()) * 1e-3) / 1e6
    if abs(recs_b[args.steps - 1].residual - rec.residual) > 1e-12 * abs(rec.residual):
        raise RuntimeError("pipelined steps disagree with the synchronous step")

    if world > 1:
        # each rank moves only its own (+ghost) points across PCIe
        n_loc = solver.owned_points
        bt = torch.tensor([n_loc * 64, n_loc * 64 + C.sizeof(rec)], device="cuda", dtype=torch.int64)
        torch.distributed.all_reduce(bt)
        h2d_b, d2h_b = int(bt[0].item()), int(bt[1].item())
    else:
        h2d_b = int(Uh.numel() * 8 + dUh.numel() * 8)
        d2h_b = int(Uo.numel() * 8 + dUo.numel() * 8 + C.sizeof(rec))

    # ---- per-kernel profile (CUDA events between launches) for the roofline
    prof = solver.profile_kernels(reps=5)
    total_ms = sum(t for _, t in prof)
    agg = {}
    for name, t in prof:
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
    flux_ms = agg["flux_residual"][1]
    ls = kf.build_ls_coefficients(cloud)
    n_s = float(sum(np.count_nonzero(ls.split_w[k]) for k in ls.split_w)) / N
    n_own = solver.owned_points  # the flux kernels of this rank's partition(s)
    flux_bytes = n_own * (FLUX_BYTES_FIXED + 4.0 * n_s)
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    if not hbm_peak:
        hbm_peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    achieved = flux_bytes / (flux_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "flux_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            if tj.get("points") == N and world == 1 and args.parts == 1:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    fp64_peak = kf.measure_fp64_peak(local)
    fp64 = None
    fpath = os.path.join(ROOT, "profiles", "flux_fp64.json")
    if os.path.exists(fpath):
        try:
            with open(fpath) as f:
                fj = json.load(f)
            if fj.get("points") == N and world == 1 and args.parts == 1:
                fl = float(fj["fp64_flops_per_launch"])
                ach = fl / (flux_ms * 1e-3) / 1e12
                fp64 = {"achieved_tflops": ach, "peak_tflops": fp64_peak, "frac": ach / fp64_peak,
                        "flops_per_launch": fl, "source": fj.get("source"),
                        "how": "ncu dfma*2 + dmul + dadd thread instructions of one launch / this run's "
                               "CUDA-event kernel time; peak = measured DFMA loop (kf_measure_fp64_peak)"}
        except Exception:
            fp64 = None

    # whole-iteration roofline: algorithmic bytes of all
    # stages, the ncu FP64 count of all 13 launches, against the step time
    n_f = float(len(cloud.nbr.ids)) / N
    iter_bytes = n_own * (ITER_BYTES_FIXED + 4.0 * (3 * n_f + 3 * n_s))
    step_s = ms_max / args.steps * 1e-3
    iteration = {"alg_bytes": iter_bytes, "achieved_gbs": iter_bytes / step_s / 1e9,
                 "hbm_frac": iter_bytes / step_s / 1e9 / hbm_peak,
                 "how": "SURVEY.md 8(d) B_alg per point (144+4nf | 2x 176+4nf | 144+4ns | 176 | 2x 121+4ns | 97) "
                        "x points / measured step time"}
    ipath = os.path.join(ROOT, "profiles", "iter_fp64.json")
    if os.path.exists(ipath) and world == 1 and args.parts == 1:
        try:
            with open(ipath) as f:
                ij = json.load(f)
            if ij.get("points") == N:
                fl = float(ij["fp64_flops_per_iteration"])
                t_ideal = max(iter_bytes / (hbm_peak * 1e9), fl / (fp64_peak * 1e12))
                iteration.update({"fp64_flops": fl, "fp64_tflops": fl / step_s / 1e12,
                                  "fp64_frac": fl / step_s / 1e12 / fp64_peak,
                                  "t_ideal_over_t": t_ideal / step_s, "fp64_source": ij.get("source")})
        except Exception:
            pass

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated NACA 0012 O-grid, deterministic; no RNG)",
        "config": {
            "workload": f"naca0012:{spec['n_wall']}:{spec['n_radial']}:20 M{spec['mach']} AoA{spec['aoa']:g} "
                        f"{spec['variant']} CFL{spec['cfl']} n_inner3, one fixed-point iteration (re-run of "
                        "iteration 6 from the resident iteration-5 state)",
            "baseline_config": args.case,
            "points": N, "colours": int(kf.color_points(cloud).n_colors),
            "parallelism": (f"domain-decomposition x{world} (angular wedges, NCCL halos)" if world > 1 else
                            f"single-gpu, {args.parts} in-process partitions" if args.parts > 1 else "single-gpu"),
            "l2": "inputs larger than L2 (per-iteration working set > 400 MB vs 126 MB L2)",
        },
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
                "call": "kf_step_host_batch (C ABI, pinned host buffers; every step H2D(U, dU_prev) + "
                        "iteration + D2H(U', dU, record), copies of neighbouring steps overlapped); "
                        "host wall clock around the call",
                "sync_value": e2e_sync_value,
                "batches": "median of 3 timed batches of `steps` steps",
                "sync_call": "kf_step_host, one blocking call per step"},
        "gpu_launches": launches,
        "clocks": clocks,
        "roofline": {
            "bound": "hbm", "kernel": "flux_residual", "achieved": achieved, "peak": hbm_peak,
            "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": traffic,
            "peak_source": peak_src,
            "algorithmic_bytes_per_launch": flux_bytes,
            "kernel_ms": flux_ms, "kernel_share_of_step": flux_ms / total_ms if total_ms else None,
            "note": "the flux kernel is FP64-pipe bound (SURVEY.md F4); see fp64",
            "fp64_peak_tflops_measured": fp64_peak,
            "fp64": fp64,
            "iteration": iteration,
        },
        "kernels_ms": {k: {"launches": v[0], "ms": v[1]} for k, v in agg.items()},
        "check": {"residual": recs[WARM_ITERS].residual if len(recs) > WARM_ITERS else None,
                  "cl": recs[WARM_ITERS].cl if len(recs) > WARM_ITERS else None,
                  "first_order_points": recs[WARM_ITERS].first_order_points if len(recs) > WARM_ITERS else None},
    }
    if rank == 0 and not args.no_cpu_baseline:
        secs, n_ref, kind = reference_cpu(8, cpu_cores(), spec)
        secs = secs[1:] or secs
        line["cpu_baseline"] = {
            "value": n_ref / float(np.median(secs)) / 1e6, "unit": UNIT, "cores": cpu_cores(),
            "kind": kind, "sample": f"{len(secs)} iterations of the same case on the host "
                                    "(median per-iteration time, warm-up iteration excluded)"}
    if rank == 0 and world == 1 and args.parts == 1 and args.case == 2:
        line["time_to_drop"] = time_to_drop(kf, 1.0, with_cpu=not args.no_cpu_baseline)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
