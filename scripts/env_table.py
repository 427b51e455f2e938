#!/usr/bin/env python
"""Table of gpurun_out/env_*.json (scripts/gpu_envs.sh): value and per-kernel us."""
import glob, json, os, sys
envs = ["default"] + (sys.argv[1].split(";") if len(sys.argv) > 1 else [])
rows = {}
for f in sorted(glob.glob("gpurun_out/env_*_*.json")):
    r, tag = os.path.basename(f)[4:-5].split("_", 1)
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    name = "default" if tag == "default" else envs[int(tag)]
    k = {n: round(v["ms"] * 1000 / v["launches"], 1) for n, v in d["kernels_ms"].items()}
    print(f"rep {r} {name:34s} {d['value']:8.1f}  {k}")
