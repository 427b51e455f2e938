#!/usr/bin/env python
"""Stall samples aggregated per CUDA source line for the kernels matching a
regex in an ncu report (needs -lineinfo): python scripts/ncu_lines.py rep regex [top]"""
import collections, csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + sys.argv[2]], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
hdr = next(r for r in rows if r and r[0] == "Line No")
si = hdr.index("Warp Stall Sampling (All Samples)")
cur, agg, src = None, collections.Counter(), {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) != len(hdr) or r[0] in ("Line No", "", "0"):
        continue
    key = (cur, int(r[0]))
    src[key] = r[1]
    try:
        agg[key] += int(r[si])
    except ValueError:
        pass
tot = sum(agg.values()) or 1
print("total samples", tot)
for k, v in agg.most_common(top):
    print(f"{v:7d} {100 * v / tot:5.1f}% {k[0]}:{k[1]} {src[k].strip()[:90]}")
