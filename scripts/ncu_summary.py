#!/usr/bin/env python
"""Summarise ncu evidence into profiles/ (run here, on the CPU box).

  python scripts/ncu_summary.py full   <report.ncu-rep> <out.json> [points]
  python scripts/ncu_summary.py launch <launches.csv>   <out.txt>
  python scripts/ncu_summary.py fp64   <fp64.csv>       <points>
  python scripts/ncu_summary.py fp64_iter <fp64_iter.csv> <points>

`full` keeps, per captured launch, duration, DRAM bytes, FP64-pipe and
occupancy metrics; with `points` it also (re)writes profiles/flux_traffic.json
(the DRAM traffic per launch of the flux-residual kernel that bench.py reports
as roofline.traffic). `launch` aggregates an ncu launch list per kernel.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
]


def to_num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return v


def full(rep, out, points=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    launches = []
    for d in data:
        rec = {"kernel": d[ki]}
        for m in KEEP:
            if m in hdr:
                i = hdr.index(m)
                rec[m] = to_num(d[i])
                if units[i]:
                    rec[m + " [unit]"] = units[i]
        launches.append(rec)
    with open(out, "w") as f:
        json.dump({"report": os.path.basename(rep), "launches": launches}, f, indent=1)
    print(f"wrote {out}: {len(launches)} launches")
    if points:
        flux = [r for r in launches if r["kernel"].startswith("void k_residual")]
        if flux:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = []
            for r in flux:
                b = 0.0
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    b += r[m] * scale.get(r.get(m + " [unit]", "byte"), 1)
                tot.append(b)
            tj = {"points": int(points), "kernel": flux[0]["kernel"],
                  "dram_bytes_per_launch": sum(tot) / len(tot), "source": os.path.basename(rep),
                  "how": "ncu --set full: dram__bytes_read.sum + dram__bytes_write.sum, mean over captured launches"}
            with open(os.path.join(ROOT, "profiles", "flux_traffic.json"), "w") as f:
                json.dump(tj, f, indent=1)
            print("flux traffic", tj)


def launch(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in data:
        n = r[ki].split("(")[0]
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list ({os.path.basename(path)}): gpu__time_duration.sum per kernel, "
                "cold-cache serialised launches -- compare SHARES\n")
        f.write(f"{'kernel':44s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}\n")
        for k, v in agg.items():
            f.write(f"{k:44s} {v[0]:8d} {v[1] / 1e3:10.1f} {v[1] / 1e3 / v[0]:9.1f} {100 * v[1] / tot:5.1f}%\n")
    print(open(out).read())


def fp64(path, points, out=None):
    """profiles/flux_fp64.json from an ncu --csv --metrics run over k_residual
    (smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on.sum)."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = collections.defaultdict(dict)
    ids = hdr.index("ID")
    for r in data:
        if "k_residual" not in r[ki]:
            continue
        per[r[ids]][r[mi]] = float(r[vi].replace(",", ""))
    launches = list(per.values())
    if not launches:
        raise SystemExit("no k_residual launches in " + path)
    def mean(m):
        return sum(l.get(m, 0.0) for l in launches) / len(launches)
    dfma = mean("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum")
    dmul = mean("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum")
    dadd = mean("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum")
    tj = {"points": int(points), "dfma": dfma, "dmul": dmul, "dadd": dadd,
          "fp64_flops_per_launch": 2 * dfma + dmul + dadd,
          "fp64_pipe_ops_per_point": (dfma + dmul + dadd) / int(points),
          "source": os.path.basename(path)}
    with open(out or os.path.join(ROOT, "profiles", "flux_fp64.json"), "w") as f:
        json.dump(tj, f, indent=1)
    print(tj)


def fp64_iter(path, points, out=None):
    """profiles/iter_fp64.json: FP64 flops (2 DFMA + DMUL + DADD) of every
    kernel of one iteration (an ncu --csv --metrics capture of 13 launches)."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, mi, vi, ids = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = collections.OrderedDict()
    for r in data:
        per.setdefault(r[ids], {"kernel": r[ki].split("(")[0]})[r[mi]] = float(r[vi].replace(",", ""))
    kern = collections.OrderedDict()
    total = 0.0
    for l in per.values():
        f = 2 * l.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0) + \
            l.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0) + \
            l.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0)
        k = kern.setdefault(l["kernel"], {"launches": 0, "fp64_flops": 0.0})
        k["launches"] += 1
        k["fp64_flops"] += f
        total += f
    tj = {"points": int(points), "launches": len(per), "fp64_flops_per_iteration": total,
          "fp64_flops_per_point": total / int(points), "kernels": kern, "source": os.path.basename(path),
          "how": "ncu smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on.sum of the 13 launches of "
                 "one iteration; flops = 2 DFMA + DMUL + DADD"}
    with open(out or os.path.join(ROOT, "profiles", "iter_fp64.json"), "w") as f:
        json.dump(tj, f, indent=1)
    print(json.dumps(tj, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "fp64_iter":
        fp64_iter(sys.argv[2], sys.argv[3])
        sys.exit(0)
    if sys.argv[1] == "fp64":
        fp64(sys.argv[2], sys.argv[3])
        sys.exit(0)
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launch(sys.argv[2], sys.argv[3])
