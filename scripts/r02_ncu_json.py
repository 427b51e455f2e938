#!/usr/bin/env python
"""Per-case ncu evidence for bench.py's rooflines (run here, on the CPU box,
over files gpurun brought back):

  python scripts/r02_ncu_json.py fp64    <fp64_iter.csv>  <case> <points>
  python scripts/r02_ncu_json.py traffic <report.ncu-rep> <case> <points>
  python scripts/r02_ncu_json.py launch  <launches.csv>   <out.txt>

fp64 -> profiles/r02_fp64_case<k>.json: FP64 flops (2 DFMA + DMUL + DADD thread
instructions) of every kernel of ONE iteration, grouped by the names
Solver.profile_kernels uses (grad_pass1, grad_passk, flux_residual,
lusgs_forward, lusgs_backward, update_bc_q, finalize).
traffic -> profiles/r02_traffic_case<k>.json: DRAM bytes (read + write) of
the same launches from an `ncu --set full` capture.
launch -> per-kernel share of the iteration from an ncu launch list.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOW_FP64 = ("ncu smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on.sum of the launches of one "
            "iteration; flops = 2 DFMA + DMUL + DADD")


def group(name):
    if "k_grad_t<1>" in name or "k_grad_t<(bool)1>" in name or "k_grad<1>" in name:
        return "grad_pass1"
    if "k_grad" in name:
        return "grad_passk"
    if "k_residual" in name:
        return "flux_residual"
    if "k_forward" in name:
        return "lusgs_forward"
    if "k_backward" in name:
        return "lusgs_backward"
    if "k_update" in name:
        return "update_bc_q"
    if "k_finalize" in name:
        return "finalize"
    return None


def _csv_rows(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    return rows[0], rows[1:]


def fp64(path, case, points):
    hdr, data = _csv_rows(path)
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    names = {}
    for d in data:
        per[d[ii]][d[mi]] += float(d[vi].replace(",", ""))
        names[d[ii]] = d[ki]
    out = collections.OrderedDict()
    total = 0.0
    for lid in sorted(per, key=int):
        g = group(names[lid])
        if g is None:
            continue
        m = per[lid]
        fl = (2 * m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
              + m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
              + m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"])
        e = out.setdefault(g, {"launches": 0, "fp64_flops": 0.0})
        e["launches"] += 1
        e["fp64_flops"] += fl
        total += fl
    res = {"case": case, "points": points, "fp64_flops_per_iteration": total,
           "fp64_flops_per_point": total / points, "kernels": out, "source": os.path.basename(path),
           "how": HOW_FP64}
    dst = os.path.join(ROOT, "profiles", f"r02_fp64_case{case}.json")
    with open(dst, "w") as f:
        json.dump(res, f, indent=1)
    print(dst, json.dumps(res)[:400])


def traffic(rep, case, points):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    ki = hdr.index("Kernel Name")
    rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    pipe = hdr.index("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") \
        if "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active" in hdr else None
    dur = hdr.index("gpu__time_duration.sum")
    units = rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    out = collections.OrderedDict()
    for d in data:
        g = group(d[ki])
        if g is None:
            continue
        b = (float(d[rd].replace(",", "")) * scale.get(units[rd], 1.0)
             + float(d[wr].replace(",", "")) * scale.get(units[wr], 1.0))
        e = out.setdefault(g, {"launches": 0, "dram_bytes": 0.0})
        e["launches"] += 1
        e["dram_bytes"] += b
        if pipe is not None:  # FP64-pipe activity, time-weighted over the launches
            t = float(d[dur].replace(",", ""))
            e["_pipe_t"] = e.get("_pipe_t", 0.0) + t * float(d[pipe].replace(",", ""))
            e["_t"] = e.get("_t", 0.0) + t
    for e in out.values():
        if "_t" in e:
            e["fp64_pipe_active_pct"] = e.pop("_pipe_t") / e.pop("_t")
    res = {"case": case, "points": points, "kernels": out, "source": os.path.basename(rep),
           "how": "ncu --set full: dram__bytes_read.sum + dram__bytes_write.sum summed over the launches of "
                  "one iteration (cold-cache, serialised replays); fp64_pipe_active_pct = "
                  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active, time-weighted"}
    dst = os.path.join(ROOT, "profiles", f"r02_traffic_case{case}.json")
    with open(dst, "w") as f:
        json.dump(res, f, indent=1)
    print(dst, json.dumps(res)[:400])


def launch(path, out):
    hdr, data = _csv_rows(path)
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    iter_keys = set()
    for d in data:
        g = group(d[ki])
        if g:
            iter_keys.add(g)
        g = g or d[ki].split("(")[0]
        a = agg.setdefault(g, [0, 0.0])
        a[0] += 1
        a[1] += float(d[vi].replace(",", "")) * 1e-3
    tot = sum(v[1] for k, v in agg.items() if k in iter_keys)
    with open(out, "w") as f:
        f.write("ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised):\n"
                "share = fraction of the per-iteration kernels' total\n")
        f.write(f"{'kernel':40s} {'launches':>8s} {'us total':>12s} {'share':>7s}\n")
        for k, (n, us) in agg.items():
            f.write(f"{k:40s} {n:8d} {us:12.1f} {us / tot if tot else 0:7.3f}\n")
    print(open(out).read())


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "fp64":
        fp64(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    elif mode == "traffic":
        traffic(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    else:
        launch(sys.argv[2], sys.argv[3])
