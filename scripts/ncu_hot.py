#!/usr/bin/env python
"""Top stall-sampled SASS lines per kernel of an ncu report (needs -lineinfo)."""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
blocks, cur = [], None
for l in raw.split("\n"):
    if l.startswith('"Kernel Name"'):
        cur = [l]
        blocks.append(cur)
    elif cur is not None:
        cur.append(l)
seen = set()
for b in blocks:
    if want not in b[0] or b[0] in seen:
        continue
    seen.add(b[0])
    rows = list(csv.reader(b[1:]))
    hdr = rows[0]
    data = [r for r in rows[1:] if len(r) == len(hdr)]
    si, src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    tot = sum(int(r[si]) for r in data) or 1
    print("=====", b[0][:90], "samples", tot)
    for r in sorted(data, key=lambda r: -int(r[si]))[:top]:
        print(f"{int(r[si]):6d} {100 * int(r[si]) / tot:5.1f}%  {r[0][-5:]} {r[src].strip()[:80]}")
