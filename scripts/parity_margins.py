#!/usr/bin/env python
"""Parity margins (GPU): for every reference-golden run case of the parity
suite, the largest relative residual-history error and the largest CL/CD
error against the reference, for the library selected by KF_LIB_PATH /
KF_FLUX_KERNEL. Prints one JSON line (the worst case) plus a table.

  python scripts/parity_margins.py [tag]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))  # tests/util imports the checkers
import paper_2406_07441_b200 as kf  # noqa: E402
from util import relmax  # noqa: E402

G = os.path.join(ROOT, "tests", "golden")
VARIANTS = ["explicit", "anandh", "anandh_ad", "manish", "manish_ad"]


def cfg(variant, **kw):
    base = dict(variant=kf.SolverVariant.parse(variant), mach_inf=0.63, aoa_deg=2.0,
                cfl=0.05 if variant == "explicit" else 0.2)
    base.update(kw)
    return kf.SolverConfig(**base)


def row(name, r, res, cl, cd):
    n = min(len(r.iters), len(res))
    return {"case": name, "iters": len(r.iters), "want_iters": int(len(res)),
            "res_rel": relmax(r.residual[:n], res[:n]),
            "clcd_abs": float(max(np.max(np.abs(r.cl[:n] - cl[:n])), np.max(np.abs(r.cd[:n] - cd[:n])))) if n else 0.0}


def main():
    rows = []
    g = np.load(os.path.join(G, "irregular_histories.npz"))
    c = kf.PointCloud.from_arrays(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["ids"])
    for v in VARIANTS:
        r = kf.Solver(c, cfg(v, n_iterations=40)).run()
        rows.append(row("irregular/" + v, r, g[v + "_residual"], g[v + "_cl"], g[v + "_cd"]))
    h = np.load(os.path.join(G, "small_histories.npz"))
    small = kf.generate_naca_ogrid("0012", 48, 12, 12.0)
    for v in VARIANTS:
        r = kf.Solver(small, cfg(v, n_iterations=60)).run()
        rows.append(row("small/" + v, r, h[v + "_residual"], h[v + "_cl"], h[v + "_cd"]))
    h1 = np.load(os.path.join(G, "config1_history.npz"))
    c1 = kf.generate_naca_ogrid("0012", 320, 120, 20.0)
    r = kf.Solver(c1, cfg("manish_ad", n_iterations=1000)).run()
    rows.append(row("config1/manish_ad", r, h1["residual"], h1["cl"], h1["cd"]))
    m = np.load(os.path.join(G, "config_matrix.npz"))
    meta = json.loads(str(m["meta"]))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_gpu_parity import _solver_config  # noqa: E402
    for name in sorted(meta):
        case = meta[name]
        if not case["iters"]:
            continue
        r = kf.Solver(kf.generate_naca_ogrid(*case["cloud"]), _solver_config(case["cfg"])).run()
        rows.append(row("matrix/" + name, r, m[name + "_residual"], m[name + "_cl"], m[name + "_cd"]))
    tag = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("KF_FLUX_KERNEL", "default")
    for x in rows:
        print(f"{x['case']:34s} iters {x['iters']:4d}/{x['want_iters']:4d}  res_rel {x['res_rel']:.2e}  "
              f"clcd_abs {x['clcd_abs']:.2e}")
    worst = max(rows, key=lambda x: x["res_rel"])
    print(json.dumps({"tag": tag, "cases": len(rows), "worst_res_rel": worst["res_rel"], "worst_case": worst["case"],
                      "worst_clcd_abs": max(x["clcd_abs"] for x in rows),
                      "iter_mismatch": [x["case"] for x in rows if x["iters"] != x["want_iters"]]}))


if __name__ == "__main__":
    main()
