#!/usr/bin/env python
"""Benchmark of the B200 implicit-LSKUM hot path (one JSON line on rank 0).

Workload (default: BASELINE.json configs[4], the largest single-GPU config,
"synthetic NACA 0012 cloud >= 40M points"): NACA 0012 O-grid 10240x3920
(40,140,800 points, radius 20), M 0.63, AoA 2 deg, modified LU-SGS with
exact-AD JVPs (manish_ad), CFL 0.2, 3 inner gradient passes, physical BCs. A
*step* is one fixed-point iteration (driver.cpp:218-276): q, 3 q-derivative
passes, split-flux residual, time step + S-term + diagonal, 4 forward and 3
backward colour sweeps, update + BCs, residual norm and CL/CD. The timed
steps are consecutive iterations of the run (after 5 + W warm-up iterations),
like the reference arm's; cases whose reference run aborts within the timed
window (configs 2 and 3) or --restart re-run iteration 6 from the resident
iteration-5 state instead (kf_bench_mode: the restart copy of U and dU_prev
inside every timed step). --case 2|3|4 selects the other BASELINE clouds.

  value : device-timed Mpoint-iter/s (CUDA events on the library stream,
          state resident in HBM), whole job over all ranks.
  e2e   : the same metric through the reference-facing C-ABI call
          kf_step_host_batch with pinned HOST buffers: H2D(U, dU_prev) +
          iteration + D2H(U', dU, record) every step; `e2e.pcie` is the
          box's own concurrent-copy ceiling for those bytes, measured in the
          same run.

Multi-GPU (--gpus N under torchrun, one process per GPU): STRONG scaling of
the same config-5 cloud, cut into N angular wedges; every rank solves its
wedge with ghost points refreshed by grouped ncclSend/ncclRecv between
dependent stages plus one ncclAllReduce of the residual/forces/abort partials
per iteration. `value` is the cloud's points times steps over the
max-over-ranks device time.

--impl reference times the reference's own CPU solver (oracle/_ref, all host
threads) on the same case and cloud; both arms print the same `config`.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs (SURVEY.md §8(d) clouds)
CASES = {
    1: dict(digits="0012", n_wall=320, n_radial=120, radius=20.0, mach=0.63, aoa=2.0, cfl=0.2,
            variant="manish_ad"),
    2: dict(digits="0012", n_wall=1280, n_radial=500, radius=20.0, mach=0.85, aoa=1.0, cfl=0.2,
            variant="manish_ad"),
    3: dict(digits="0012", n_wall=2560, n_radial=960, radius=20.0, mach=1.2, aoa=0.0, cfl=0.2,
            variant="anandh_ad"),
    4: dict(digits="0012", n_wall=5120, n_radial=1920, radius=20.0, mach=0.63, aoa=2.0, cfl=0.2,
            variant="manish_ad"),
    5: dict(digits="0012", n_wall=10240, n_radial=3920, radius=20.0, mach=0.63, aoa=2.0, cfl=0.2,
            variant="manish_ad"),
}
DEFAULT_CASE = 5
METRIC = "Mpoint-iter/s (FP64 LU-SGS+AD) and time-to-residual-drop, NACA 0012 clouds"
UNIT = "Mpoint-iter/s"
WARM_ITERS = 5
E2E_MIN_STEPS = 64  # steps per pipelined host-fed call (see the e2e section)
# reference arm: iterations timed per run (13 s each on config 5 at 16 cores),
# so the whole arm (46 s of reference setup included) ends in ~3 minutes
REF_MAX_STEPS = 8
# SURVEY.md §8(d) algorithmic bytes per point (FP64 = 8 B, index = 4 B,
# neighbour gathers counted as cache hits):
FLUX_BYTES_FIXED = 144.0     # S3: q 32 + qx,qy 64 + xy 16 + R 32 (+ 4 n_s ids)
GRAD1_BYTES_FIXED = 144.0    # S1: U 32 + xy 16 + q 32 + qx,qy 64 (+ 4 n_f)
GRADK_BYTES_FIXED = 176.0    # S2: q 32 + qx,qy 64 + xy 16 + qx,qy 64 (+ 4 n_f)
SWEEP_BYTES_FIXED = 176.0 + 2 * 121.0  # S4 (dt, d, S) + S5 + S6 (+ 2 x 4 n_s)
ITER_BYTES_FIXED = 1155.0    # 144 + 2x176 + 144 + 176 + 121 + 121 + 97


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region through
    NVML (every 2 ms); nvidia-smi as the fallback."""

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
        while True:
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            if self._stop.wait(0.002):
                break

    def _smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "sw_thermal_slowdown", "hw_thermal_slowdown", "sw_power_cap"]
        while True:
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
            if self._stop.wait(0.05):
                break

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


def gpu_local_cpus(index):
    """Host cores on the GPU's NUMA node (nvmlDeviceGetCpuAffinity), or None."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= set(os.sched_getaffinity(0))
        return cpus or None
    except Exception:
        return None


def workload_of(spec):
    return (f"naca0012:{spec['n_wall']}:{spec['n_radial']}:{spec['radius']:g} M{spec['mach']} "
            f"AoA{spec['aoa']:g} {spec['variant']} CFL{spec['cfl']} n_inner3, one fixed-point iteration")


def config_of(spec, case, n, colours):
    """The `config` object both arms print (identical for the same case)."""
    return {"workload": workload_of(spec), "baseline_config": case, "points": int(n),
            "colours": int(colours),
            "l2": "inputs larger than L2 (per-iteration working set > 400 MB vs 126 MB L2)"}


def spec_for(case, points=None):
    spec = dict(CASES[case])
    if points:
        nw, nr = points.split(":")
        spec["n_wall"], spec["n_radial"] = int(nw), int(nr)
    return spec


def _refpy():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refpy  # checker: only the cpu_baseline / reference arm may use it
    return refpy


def reference_sample(spec, n_timed, threads, warm=1):
    """The reference solver (oracle/_ref, else the C restatement) on the case:
    setup seconds, per-iteration seconds of iterations warm+1..warm+n_timed
    (runs restarted from freestream before the reference's own aborts, the
    first `warm` iterations of every run excluded), N, colours, kind."""
    refpy = _refpy()
    kind = "reference" if refpy.ref_available() else "port"
    t0 = time.perf_counter()
    if kind == "reference":
        refpy.Reference.num_threads(threads)
        ctx = refpy.Reference.generate(spec["digits"], spec["n_wall"], spec["n_radial"], spec["radius"])
        colours = int(ctx.colors().max())
    else:
        os.environ["OMP_NUM_THREADS"] = str(threads)
        import paper_2406_07441_b200 as kf
        c = kf.generate_naca_ogrid(spec["digits"], spec["n_wall"], spec["n_radial"], spec["radius"])
        nb = c.nbr
        ctx = refpy.Oracle(c.x, c.y, c.kind, c.normal_x, c.normal_y, nb.offsets, nb.ids)
        colours = int(kf.color_points(c).n_colors)
    setup = time.perf_counter() - t0
    secs = []
    while len(secs) < n_timed:
        m = min(n_timed - len(secs) + warm, 20)
        t1 = time.perf_counter()
        r = ctx.run(variant=spec["variant"], n_iterations=m, mach=spec["mach"], aoa_deg=spec["aoa"],
                    cfl=spec["cfl"])
        wall = time.perf_counter() - t1
        s = (list(r.seconds[warm:]) if kind == "reference" else
             [wall / max(len(r.residual), 1)] * max(len(r.residual) - warm, 0))
        if not s:
            break
        secs.extend(s)
    n = ctx.n
    del ctx
    return setup, secs[:n_timed], n, colours, kind


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = cpu_cores()
    spec = spec_for(args.case, args.points)
    k = max(1, min(args.steps, REF_MAX_STEPS))
    warm = min(args.warmup, 3)  # (W >= 3 warm-up steps, bounded: 13 s each on config 5)
    setup, secs, n, colours, kind = reference_sample(spec, k, threads, warm)
    total = float(np.sum(secs))
    value = n * len(secs) / total / 1e6
    sample = (f"{len(secs)} reference iterations of the same case and cloud (run_fixed_point through the "
              f"reference's own API; the run's first {warm} iterations excluded as warm-up; at most "
              f"{REF_MAX_STEPS} timed so the arm ends in minutes: the reference iteration is "
              f"{total / len(secs):.1f} s)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(secs), "warmup": warm, "ms_per_step": 1e3 * total / len(secs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (generated NACA 0012 O-grid, deterministic; no RNG)",
        "config": config_of(spec, args.case, n, colours),
        "parallelism": f"cpu-openmp ({threads} host threads)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_setup_seconds": setup,
    }
    print(json.dumps(line), flush=True)
    return 0


class PinnedPool:
    """Page-locked host buffers for the e2e copies: anonymous mmaps with
    transparent huge pages, first touched by the filling copy and registered
    with cudaHostRegister (2 MB pages: fewer IOMMU / page-table entries per
    DMA; ~2-3 % more concurrent H2D+D2H than cudaHostAlloc's buffers on the
    B200 box, profiles/r02_pcie_probe2.txt, and ~10x faster to pin).
    torch.pin_memory() if registration fails."""

    def __init__(self, torch):
        self.torch = torch
        self.rt = torch.cuda.cudart()
        self.held = []

    def empty(self, shape, src=None):
        import mmap
        torch = self.torch
        nb = int(np.prod(shape)) * 8
        try:
            m = mmap.mmap(-1, max(nb, 8), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
            if hasattr(mmap, "MADV_HUGEPAGE"):
                m.madvise(mmap.MADV_HUGEPAGE)
            t = torch.frombuffer(m, dtype=torch.float64, count=int(np.prod(shape))).view(*shape)
            if src is not None:
                t.copy_(torch.from_numpy(np.ascontiguousarray(src)))
            else:
                t.zero_()
            if int(self.rt.cudaHostRegister(t.data_ptr(), nb, 0)) != 0:
                raise RuntimeError("cudaHostRegister")
            self.held.append((t, m))
            return t
        except Exception:
            t = torch.from_numpy(np.ascontiguousarray(src)) if src is not None else torch.empty(shape, dtype=torch.float64)
            return t.pin_memory()

    def release(self):
        for t, m in self.held:
            self.rt.cudaHostUnregister(t.data_ptr())
        self.held = []


def pcie_ceiling(torch, n, step_ms, reps=5, rounds=4, hin=None, hout=None):
    """The box's concurrent host<->device copy ceiling for one e2e step's
    bytes: H2D of (U, dU_prev) and D2H of (U', dU) on two streams, from and to
    pinned buffers of the step's size (the e2e's own buffers when given),
    `rounds` steps' worth back to back per timing (the sustained rate a
    pipelined run sees, not one cold burst), timed with events (best of
    `reps`)."""
    dev = torch.device("cuda")
    pool = PinnedPool(torch)  # (the e2e's kind of buffer)
    if hin is None:
        hin = [pool.empty((n, 4)) for _ in range(2)]
    if hout is None:
        hout = [pool.empty((n, 4)) for _ in range(2)]
    din = [torch.empty((n, 4), dtype=torch.float64, device=dev) for _ in range(2)]
    dout = [torch.empty((n, 4), dtype=torch.float64, device=dev) for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    best = {}
    for mode in ("h2d", "d2h", "both"):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream())
            s_in.wait_event(e0)
            s_out.wait_event(e0)
            for _ in range(rounds):
                if mode in ("h2d", "both"):
                    with torch.cuda.stream(s_in):
                        for a, b in zip(din, hin):
                            a.copy_(b, non_blocking=True)
                if mode in ("d2h", "both"):
                    with torch.cuda.stream(s_out):
                        for a, b in zip(hout, dout):
                            a.copy_(b, non_blocking=True)
            e1.record(s_in)
            e2.record(s_out)
            torch.cuda.synchronize()
            ts.append(max(e0.elapsed_time(e1), e0.elapsed_time(e2)) / rounds)
        best[mode] = min(ts)
    del hin, hout
    pool.release()
    bytes_dir = 2 * n * 32
    both = best["both"]
    return {"h2d_gbs": bytes_dir / best["h2d"] / 1e6, "d2h_gbs": bytes_dir / best["d2h"] / 1e6,
            "concurrent_ms_per_step": both,
            "bound_value": n / (max(both, step_ms) * 1e-3) / 1e6,
            "how": f"bare H2D of 2 x (n, 4) f64 and D2H of 2 x (n, 4) f64 per step on two streams from/to "
                   f"pinned buffers (the e2e's), {rounds} steps back to back per timing (best of {reps}); bound = points / "
                   "max(copy time per step, device step time)"}


def profiles_for(case, name):
    """Committed per-case ncu evidence (profiles/r02_<name>_case<k>.json)."""
    path = os.path.join(ROOT, "profiles", f"r02_{name}_case{case}.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def time_to_drop_c1(kf, with_cpu=True, decades=1.0):
    """North-star time to a fixed residual drop (RunHistory::iterations_to_decades,
    driver.cpp:169-178) on BASELINE config 1 (NACA 0012 320x120, M 0.63,
    AoA 2, manish_ad, CFL 0.2): the reference reaches ~1 decade before its
    abort in iteration 423. GPU: device seconds of the
    iterations up to the drop (per-iteration globaltimer records). CPU: the
    reference's own per-iteration seconds for the same iterations, all host
    threads. Also the drop-in wall clock of the whole run, setup included
    (generate + kf_create + kf_run vs generate + run_fixed_point)."""
    spec = CASES[1]
    cfg = kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2,
                          n_iterations=1000)
    # (the process's one-time CUDA context / module load, ~2.4 s, and the
    # first use of this cloud size's kernels are paid by a warm-up solve of
    # the same case first: the drop-in figure is a steady caller's)
    kf.Solver(kf.generate_naca_ogrid("0012", spec["n_wall"], spec["n_radial"], spec["radius"]), cfg).run()
    w0 = time.perf_counter()
    c = kf.generate_naca_ogrid("0012", spec["n_wall"], spec["n_radial"], spec["radius"])
    s = kf.Solver(c, cfg)
    h = s.run(want_state=True)
    gpu_wall = time.perf_counter() - w0
    h = s.run(want_state=False)  # warm (graphs, caches) for the device timing
    k = h.iterations_to_decades(decades)
    out = {"config": workload_of(spec).replace(", one fixed-point iteration", "") + ", 1000 iterations",
           "baseline_config": 1, "decades": decades, "iterations": k, "recorded_iterations": len(h.iters),
           "abort": h.abort_reason}
    if k > 0:
        out["gpu_seconds"] = float(sum(r.seconds for r in h.iters[:k]))
    drop = {"gpu_wall_seconds": gpu_wall,
            "gpu_call": "generate_naca_ogrid + Solver (kf_create) + run (kf_run, 1000 iterations: "
                        f"{len(h.iters)} recorded + abort) + final state download, host wall clock; the "
                        "process's one-time CUDA context and module load (~2.4 s, profiles/"
                        "r02_ab_grad_minb_and_dropin.txt) excluded by a warm-up solve of the same case"}
    if with_cpu:
        refpy = _refpy()
        if refpy.ref_available():
            refpy.Reference.num_threads(cpu_cores())
            w0 = time.perf_counter()
            ref = refpy.Reference.generate("0012", spec["n_wall"], spec["n_radial"], spec["radius"])
            r = ref.run(variant="manish_ad", n_iterations=1000, mach=0.63, aoa_deg=2.0, cfl=0.2)
            drop["cpu_wall_seconds"] = time.perf_counter() - w0
            drop["cpu_call"] = "Reference.generate + run_fixed_point (1000 iterations), host wall clock"
            drop["speedup"] = drop["cpu_wall_seconds"] / gpu_wall
            drop["same_history"] = bool(len(r.residual) == len(h.iters) and r.abort_reason == h.abort_reason)
            if k > 0:
                out["cpu_seconds"] = float(np.sum(r.seconds[:k]))
                out["cpu_kind"] = "reference"
                out["cpu_cores"] = cpu_cores()
                out["speedup"] = out["cpu_seconds"] / out["gpu_seconds"]
    out["dropin_whole_run"] = drop
    return out


def time_to_drop_c4(kf, with_cpu=True, max_iters=3000):
    """Time to the residual drop actually reached on BASELINE config 4
    (NACA 0012 5120x1920 = 9.8M points, M 0.63, AoA 2, manish_ad, CFL 0.2):
    10 decades are unreachable, so the run goes `max_iters`
    iterations (or to its abort), the reached drop is rounded down to 0.1
    decade, and the time is that of the iterations up to it
    (iterations_to_decades, driver.cpp:169-178). CPU: the reference's measured
    per-iteration time on the same cloud (median of 2 sampled iterations) x
    the same iteration count -- extrapolated, since thousands of 3.3-s
    reference iterations do not fit a bench run."""
    spec = CASES[4]
    cfg = kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=spec["mach"], aoa_deg=spec["aoa"],
                          cfl=spec["cfl"], n_iterations=max_iters)
    c = kf.generate_naca_ogrid("0012", spec["n_wall"], spec["n_radial"], spec["radius"])
    s = kf.Solver(c, cfg)
    h = s.run(want_state=False)
    res = h.residual
    out = {"config": workload_of(spec).replace(", one fixed-point iteration", "") + f", {max_iters} iterations",
           "baseline_config": 4, "points": c.n(), "recorded_iterations": len(h.iters),
           "abort": h.abort_reason or None}
    del s
    if len(res) < 2 or not res[0] > 0:
        return out
    reached = float(np.log10(res[0] / np.min(res)))
    dec = float(np.floor(reached * 10.0) / 10.0)
    out["decades_reached"] = reached
    out["decades"] = dec
    k = h.iterations_to_decades(dec) if dec > 0 else 0
    out["iterations"] = k
    if k > 0:
        out["gpu_seconds"] = float(sum(r.seconds for r in h.iters[:k]))
        if with_cpu:
            setup, secs, n, _, kind = reference_sample(spec, 2, cpu_cores())
            per_it = float(np.median(secs))
            out.update({"cpu_seconds": per_it * k, "cpu_seconds_per_iteration": per_it, "cpu_kind": kind,
                        "cpu_cores": cpu_cores(), "cpu_how": f"extrapolated: {k} x the median of {len(secs)} "
                        "measured reference iterations on the same cloud",
                        "speedup": per_it * k / out["gpu_seconds"]})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip time-to-drop and drop-in legs")
    ap.add_argument("--profile-only", action="store_true",
                    help="run a few steps for ncu (no JSON line)")
    ap.add_argument("--points", default=None, help="override cloud n_wall:n_radial")
    ap.add_argument("--parts", type=int, default=1, help="in-process partitions on one GPU")
    ap.add_argument("--variant", default=None,
                    choices=["explicit", "anandh", "anandh_ad", "manish", "manish_ad"],
                    help="override the case's solver variant (evidence runs)")
    ap.add_argument("--ordering", type=int, default=1, choices=[0, 1, 2],
                    help="in-colour point order: 0 natural, 1 Morton (default), 2 reverse Cuthill-McKee")
    ap.add_argument("--restart", action="store_true",
                    help="time re-runs of iteration 6 from the iteration-5 state (bench mode) instead of "
                         "consecutive iterations")
    ap.add_argument("--case", type=int, default=DEFAULT_CASE, choices=sorted(CASES),
                    help=f"BASELINE.json config whose cloud/case to time (default {DEFAULT_CASE})")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        return run_reference_arm(args)

    rank, world, local = dist_env()
    lw = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    if lw > 1 and (os.environ.get("OMP_NUM_THREADS") in (None, "1") and "KF_KEEP_OMP" not in os.environ):
        # the ranks of a node build their partitions concurrently: split the
        # host cores between them (torchrun's default of ONE thread per rank
        # would make the 40M-point setup ~10x slower), set before the OpenMP
        # runtime starts, i.e. before torch / the library load
        ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or lw)
        os.environ["OMP_NUM_THREADS"] = str(max(1, ncpu // lw))
    import torch
    import paper_2406_07441_b200 as kf

    # KF_BENCH_TRANSPORT=host (a test mode, never the default): the ranks
    # exchange halos through the host-staged transport over gloo and may
    # share one GPU, so the whole N > 1 bench path runs on a one-GPU box
    # (NCCL refuses two ranks on one device)
    host_tr = world > 1 and os.environ.get("KF_BENCH_TRANSPORT") == "host"
    if host_tr:
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if host_tr:
            dist.init_process_group("gloo")
        else:
            if rank == 0:
                # NCCL's communicator lines (nranks, NVLS / P2P transports) on
                # rank 0's stderr, so the run's topology can be checked
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,GRAPH")
                os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec = spec_for(args.case, args.points)
    if args.variant:
        spec["variant"] = args.variant

    t_setup = time.perf_counter()
    cloud = kf.generate_naca_ogrid(spec["digits"], spec["n_wall"], spec["n_radial"], spec["radius"])
    t_gen = time.perf_counter() - t_setup
    N = cloud.n()
    colours = int(kf.color_points(cloud).n_colors)
    # consecutive iterations unless the reference's own run aborts inside the
    # window (configs 2 / 3 abort in iterations 22 / 7; the M 0.63 clouds
    # run >= 116 iterations, profiles/r02_c4_fullrun.json)
    n_window = WARM_ITERS + args.warmup + args.steps + 8
    trajectory = not args.restart and args.case in (1, 4, 5) and n_window <= 100
    cfg = kf.SolverConfig(variant=kf.SolverVariant.parse(spec["variant"]), mach_inf=spec["mach"],
                          aoa_deg=spec["aoa"], cfl=spec["cfl"], n_iterations=max(64, n_window), device=local,
                          ordering=args.ordering)
    t_create = time.perf_counter()
    if host_tr:
        def exchange(msgs):
            reqs = []
            for peer, is_send, buf in msgs:
                t = torch.from_numpy(buf)
                reqs.append(torch.distributed.isend(t, peer) if is_send else torch.distributed.irecv(t, peer))
            for r in reqs:
                r.wait()

        def allreduce(buf):
            torch.distributed.all_reduce(torch.from_numpy(buf))

        solver = kf.Solver.for_rank_host(cloud, cfg, world, rank, exchange, allreduce)
    elif world > 1:
        ids = [kf.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(ids, src=0)
        solver = kf.Solver.for_rank(cloud, cfg, world, rank, ids[0])
    else:
        solver = kf.Solver(cloud, cfg, n_parts=args.parts)
    t_create = time.perf_counter() - t_create
    solver.reset()
    solver.iterate_async(WARM_ITERS)
    recs, st = solver.sync_records()
    assert st.code == 0 and len(recs) == WARM_ITERS, st.reason
    # the resident iteration-5 state: every timed step (device and e2e) runs
    # iteration 6 from it
    U0, dU0 = solver.get_state(with_dU=True)
    if not trajectory:
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
    if world > 1:
        torch.distributed.barrier()
    ms = t0.elapsed_time(t1)
    recs, st = solver.sync_records()
    if st.code != 0:
        raise RuntimeError("benchmark iteration failed: " + st.reason.decode())
    red_dev = "cpu" if host_tr else "cuda"  # (gloo reduces host tensors)
    ms_t = torch.tensor([ms], device=red_dev)
    if world > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = N * args.steps / (ms_max * 1e-3) / 1e6  # N: points of the whole (all-rank) cloud
    launches = solver.launches_per_iteration * args.steps
    step_ms = ms_max / args.steps

    # ---- end to end through the C ABI with pinned host buffers (allocated
    # with the process on the GPU's NUMA node, so the pinned pages are local)
    full_aff = os.sched_getaffinity(0)
    local_cpus = gpu_local_cpus(local)
    if local_cpus:
        os.sched_setaffinity(0, local_cpus)
    pool = PinnedPool(torch)
    Uh = pool.empty(U0.shape, U0)
    dUh = pool.empty(dU0.shape, dU0)
    Uo = pool.empty(U0.shape)
    dUo = pool.empty(dU0.shape)
    del U0, dU0
    from paper_2406_07441_b200 import _lib
    rec = _lib.IterRecord()
    h = solver._h

    def e2e_step():
        s = _lib.lib.kf_step_host(h, C.c_void_p(Uh.data_ptr()), C.c_void_p(dUh.data_ptr()),
                                  C.c_void_p(Uo.data_ptr()), C.c_void_p(dUo.data_ptr()), C.byref(rec))
        if s.code != 0:
            raise RuntimeError(s.reason.decode())

    n_sync = min(args.steps, 8)
    for _ in range(min(args.warmup, 3)):
        e2e_step()
    torch.cuda.synchronize()
    # synchronous form: one blocking C-ABI call per step
    w0 = time.perf_counter()
    for _ in range(n_sync):
        e2e_step()
    torch.cuda.synchronize()
    sync_ms = 1e3 * (time.perf_counter() - w0) / n_sync
    # pipelined form (kf_step_host_batch): the same steps, H2D of step k+1 and
    # D2H of step k-1 on the copy engines while step k computes
    Uos = [pool.empty(tuple(Uh.shape)) for _ in range(2)]
    dUos = [pool.empty(tuple(dUh.shape)) for _ in range(2)]
    # steps per pipelined call: the pipeline's fill and drain (the first
    # step's H2D, the last one's D2H: ~2 PCIe-bound step times) amortised
    # over at least E2E_MIN_STEPS steps, as a host feeding a long run would
    m_e2e = max(args.steps, E2E_MIN_STEPS)
    recs_b = (_lib.IterRecord * m_e2e)()

    def batch(m):
        P = C.c_void_p * m
        s = _lib.lib.kf_step_host_batch(h, m, P(*[Uh.data_ptr()] * m), P(*[dUh.data_ptr()] * m),
                                        P(*[Uos[k & 1].data_ptr() for k in range(m)]),
                                        P(*[dUos[k & 1].data_ptr() for k in range(m)]), recs_b)
        if s.code != 0:
            raise RuntimeError(s.reason.decode())

    batch(min(args.warmup, 3))
    torch.cuda.synchronize()
    # host wall clock around the blocking batch call; the median of three
    # batches (the PCIe-bound step varies by several % from run to run)
    walls = []
    for _ in range(3):
        w0 = time.perf_counter()
        batch(m_e2e)
        torch.cuda.synchronize()
        walls.append(1e3 * (time.perf_counter() - w0))
    e2e_ms = float(np.median(walls))
    et = torch.tensor([e2e_ms, sync_ms * m_e2e], device=red_dev)
    if world > 1:
        torch.distributed.all_reduce(et, op=torch.distributed.ReduceOp.MAX)
    e2e_value = N * m_e2e / (float(et[0].item()) * 1e-3) / 1e6
    e2e_sync_value = N * m_e2e / (float(et[1].item()) * 1e-3) / 1e6
    if abs(recs_b[m_e2e - 1].residual - rec.residual) > 1e-12 * abs(rec.residual):
        raise RuntimeError("pipelined steps disagree with the synchronous step")
    if world > 1:
        # each rank moves only its own (+ghost) points across PCIe
        n_loc = solver.owned_points
        bt = torch.tensor([n_loc * 64, n_loc * 64 + C.sizeof(rec)], device=red_dev, dtype=torch.int64)
        torch.distributed.all_reduce(bt)
        h2d_b, d2h_b = int(bt[0].item()), int(bt[1].item())
    else:
        h2d_b = int(Uh.numel() * 8 + dUh.numel() * 8)
        d2h_b = int(Uo.numel() * 8 + dUo.numel() * 8 + C.sizeof(rec))
    # the box's copy ceiling, timed on the same pinned pages
    # (a rank moves only its owned points: the host arrays are whole-cloud
    # sized, a prefix of that many rows stands in for them)
    nl = solver.owned_points if world > 1 else N
    pcie = pcie_ceiling(torch, nl, step_ms, hin=[Uh[:nl], dUh[:nl]], hout=[Uo[:nl], dUo[:nl]])
    del Uos, dUos, Uh, dUh, Uo, dUo
    pool.release()
    pcie["frac"] = e2e_value / world / pcie["bound_value"] if world > 1 else e2e_value / pcie["bound_value"]
    if local_cpus:
        os.sched_setaffinity(0, full_aff)
    torch.cuda.empty_cache()

    # ---- per-kernel profile (CUDA events between launches) for the roofline
    prof = solver.profile_kernels(reps=3)
    total_ms = sum(t for _, t in prof)
    agg = {}
    for name, t in prof:
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
    kms = lambda k: agg.get(k, [0, 0.0])[1]
    ls = kf.build_ls_coefficients(cloud)
    n_s = float(sum(np.count_nonzero(ls.split_w[k]) for k in ls.split_w)) / N
    n_f = float(len(cloud.nbr.ids)) / N
    del ls
    n_own = solver.owned_points
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    if not hbm_peak:
        hbm_peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    fp64_peak = kf.measure_fp64_peak(local)
    single = world == 1 and args.parts == 1
    fpj = profiles_for(args.case, "fp64") if single else None   # ncu FP64 flops per kernel
    trj = profiles_for(args.case, "traffic") if single else None  # ncu DRAM bytes per kernel

    def kernel_roof(name, bytes_pp, launches_key):
        ms_k = kms(launches_key)
        if ms_k <= 0:
            return None
        alg = n_own * bytes_pp
        o = {"kernel_ms": ms_k, "launches": agg[launches_key][0], "algorithmic_bytes": alg,
             "achieved_gbs": alg / (ms_k * 1e-3) / 1e9, "hbm_frac": alg / (ms_k * 1e-3) / 1e9 / hbm_peak,
             "share_of_step": ms_k / total_ms if total_ms else None}
        if fpj and fpj.get("points") == N and launches_key in fpj.get("kernels", {}):
            fl = float(fpj["kernels"][launches_key]["fp64_flops"])
            o.update({"fp64_flops": fl, "fp64_tflops": fl / (ms_k * 1e-3) / 1e12,
                      "fp64_frac": fl / (ms_k * 1e-3) / 1e12 / fp64_peak})
        if trj and trj.get("points") == N and launches_key in trj.get("kernels", {}):
            o["traffic"] = float(trj["kernels"][launches_key]["dram_bytes"])
            o["traffic_over_alg"] = o["traffic"] / alg
            if "fp64_pipe_active_pct" in trj["kernels"][launches_key]:
                o["fp64_pipe_active_pct_ncu"] = trj["kernels"][launches_key]["fp64_pipe_active_pct"]
        return o

    flux = kernel_roof("flux_residual", FLUX_BYTES_FIXED + 4.0 * n_s, "flux_residual")
    fw = kernel_roof("lusgs_forward", 176.0 + 121.0 + 4.0 * n_s, "lusgs_forward")
    bw = kernel_roof("lusgs_backward", 121.0 + 4.0 * n_s, "lusgs_backward")
    g1 = kernel_roof("grad_pass1", GRAD1_BYTES_FIXED + 4.0 * n_f, "grad_pass1")
    gk = kernel_roof("grad_passk", 2 * (GRADK_BYTES_FIXED + 4.0 * n_f), "grad_passk")
    sweeps = None
    if fw and bw:
        sms = fw["kernel_ms"] + bw["kernel_ms"]
        alg = fw["algorithmic_bytes"] + bw["algorithmic_bytes"]
        sweeps = {"kernels": "k_forward x C (time step + S-term + diagonal + forward colour + hoisted JVP) "
                             "+ k_backward x (C-1)",
                  "kernel_ms": sms, "algorithmic_bytes": alg,
                  "bytes_per_point": "176 + 2 x (121 + 4 n_s) (SURVEY.md 8(d) S4 + S5 + S6)",
                  "achieved_gbs": alg / (sms * 1e-3) / 1e9, "hbm_frac": alg / (sms * 1e-3) / 1e9 / hbm_peak,
                  "forward": fw, "backward": bw}
        if "fp64_flops" in fw and "fp64_flops" in bw:
            fl = fw["fp64_flops"] + bw["fp64_flops"]
            sweeps.update({"fp64_flops": fl, "fp64_tflops": fl / (sms * 1e-3) / 1e12,
                           "fp64_frac": fl / (sms * 1e-3) / 1e12 / fp64_peak})
        if "traffic" in fw and "traffic" in bw:
            sweeps["traffic"] = fw["traffic"] + bw["traffic"]
            sweeps["traffic_over_alg"] = sweeps["traffic"] / alg

    iter_bytes = n_own * (ITER_BYTES_FIXED + 4.0 * (3 * n_f + 3 * n_s))
    step_s = step_ms * 1e-3
    iteration = {"alg_bytes": iter_bytes, "achieved_gbs": iter_bytes / step_s / 1e9,
                 "hbm_frac": iter_bytes / step_s / 1e9 / hbm_peak,
                 "how": "SURVEY.md 8(d) B_alg per point (144+4nf | 2x 176+4nf | 144+4ns | 176 | 2x 121+4ns | 97) "
                        "x points / measured step time"}
    if fpj and fpj.get("points") == N:
        fl = float(fpj["fp64_flops_per_iteration"])
        t_ideal = max(iter_bytes / (hbm_peak * 1e9), fl / (fp64_peak * 1e12))
        iteration.update({"fp64_flops": fl, "fp64_tflops": fl / step_s / 1e12,
                          "fp64_frac": fl / step_s / 1e12 / fp64_peak,
                          "t_ideal_over_t": t_ideal / step_s})

    roofline = {
        "bound": "hbm", "kernel": "flux_residual (k_residual_t)", "achieved": flux["achieved_gbs"],
        "peak": hbm_peak, "unit": "GB/s", "frac": flux["hbm_frac"], "traffic": flux.get("traffic"),
        "peak_source": peak_src,
        "algorithmic_bytes_per_launch": flux["algorithmic_bytes"],
        "bytes_per_point": f"144 + 4 n_s = {FLUX_BYTES_FIXED + 4 * n_s:.1f} (SURVEY.md 8(d) S3)",
        "kernel_ms": flux["kernel_ms"], "kernel_share_of_step": flux["share_of_step"],
        "note": "the flux kernel is FP64-pipe bound (SURVEY.md 8(d): ~3.8k FP64 ops per 208 B); its binding "
                "roofline is `fp64`",
        "fp64": ({"achieved_tflops": flux["fp64_tflops"], "peak_tflops": fp64_peak, "frac": flux["fp64_frac"],
                  "flops_per_launch": flux["fp64_flops"],
                  "pipe_active_pct_ncu": flux.get("fp64_pipe_active_pct_ncu"),
                  "how": "ncu 2 DFMA + DMUL + DADD thread instructions of one launch "
                         f"(profiles/r02_fp64_case{args.case}.json) / this run's CUDA-event kernel time; "
                         "peak = measured DFMA loop (kf_measure_fp64_peak). The kernel's FP64 instruction "
                         "count falls with every algorithmic saving (erf polynomial, log-free density), so "
                         "the pipe activity (ncu, pipe_active_pct_ncu) is the utilisation measure"}
                 if flux and "fp64_flops" in flux else None),
        "fp64_peak_tflops_measured": fp64_peak,
        "sweeps": sweeps,
        "gradients": {"pass1": g1, "passk": gk},
        "iteration": iteration,
    }

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated NACA 0012 O-grid, deterministic; no RNG)",
        "config": config_of(spec, args.case, N, colours),
        "parallelism": (f"domain decomposition x{world} (angular wedges, "
                        f"{'host-staged gloo halos: TEST transport' if host_tr else 'NCCL halos'}), same cloud at every N"
                        if world > 1 else f"single-gpu, {args.parts} in-process partitions" if args.parts > 1
                        else "single-gpu"),
        "step": (f"consecutive iterations {WARM_ITERS + args.warmup + 1}..{WARM_ITERS + args.warmup + args.steps} "
                 "of the run (state resident in HBM)" if trajectory else
                 "iteration 6 re-run from the resident iteration-5 state (restart copy inside the step)"),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
                "call": "kf_step_host_batch (C ABI, pinned host buffers; every step H2D(U, dU_prev) + "
                        "iteration + D2H(U', dU, record), copies of neighbouring steps overlapped); "
                        "host wall clock around the call",
                "batches": f"median of 3 timed calls of {m_e2e} steps each (max(steps, {E2E_MIN_STEPS}): the "
                           "pipeline fill and drain, ~2 step times, amortised as in a long host-fed run)",
                "sync_value": e2e_sync_value, "sync_call": f"kf_step_host, one blocking call per step "
                                                           f"({n_sync} steps)",
                "pcie": pcie,
                "numa": ({"gpu_local_cpus": len(local_cpus), "host_cpus": len(full_aff)} if local_cpus else None)},
        "gpu_launches": launches,
        "clocks": clocks,
        "roofline": roofline,
        "kernels_ms": {k: {"launches": v[0], "ms": v[1]} for k, v in agg.items()},
        "setup_seconds": {"generate": t_gen, "create": t_create},
        "check": {"residual": recs[WARM_ITERS].residual if len(recs) > WARM_ITERS else None,
                  "cl": recs[WARM_ITERS].cl if len(recs) > WARM_ITERS else None,
                  "first_order_points": recs[WARM_ITERS].first_order_points if len(recs) > WARM_ITERS else None},
    }
    del solver, cloud
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # (the contract: rank 0 at N = 1 only)
        setup, secs, n_ref, _, kind = reference_sample(spec, 1, cpu_cores())
        line["cpu_baseline"] = {
            "value": n_ref * len(secs) / float(np.sum(secs)) / 1e6, "unit": UNIT, "cores": cpu_cores(),
            "kind": kind, "sample": f"{len(secs)} reference iteration(s) of the same case and cloud on the "
                                    "host (iteration 2 of a run; iteration 1 excluded as warm-up)",
            "setup_seconds": setup}
    if rank == 0 and single and not args.no_extras:
        line["time_to_drop"] = time_to_drop_c1(kf, with_cpu=not args.no_cpu_baseline)
        if args.case in (4, 5):
            line["time_to_drop_config4"] = time_to_drop_c4(kf, with_cpu=not args.no_cpu_baseline)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
