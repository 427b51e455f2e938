"""Golden fixture on an IRREGULAR cloud, from the UNMODIFIED reference.

    python tests/golden/make_irregular.py     (build container: needs oracle/_ref)

A NACA 0012 O-grid whose interior points are jittered and given random extra
neighbours from their 5x5 index neighbourhood (degrees 5..24, irregular
greedy colouring, line/irregular LS classes), loaded through the reference's
PointCloud-from-arrays path. Stores the cloud arrays and, per variant, the
reference's 40-iteration residual/CL/CD/first-order history and final state.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from refpy import Reference  # noqa: E402

import paper_2406_07441_b200 as kf  # noqa: E402  (only to read the base O-grid arrays)


def irregular_cloud(n_wall=48, n_radial=12, radius=12.0, seed=11):
    c = kf.generate_naca_ogrid("0012", n_wall, n_radial, radius)
    rng = np.random.default_rng(seed)
    x0, y0 = c.x.copy(), c.y.copy()
    kind = c.kind.astype(np.int32)
    nb = c.nbr
    n = c.n()
    jit = np.zeros((n, 2))
    extra = [[] for _ in range(n)]
    for p in range(n):
        j, i = divmod(p, n_wall)
        if kind[p] != 1 or j < 2 or j > n_radial - 3:
            continue
        h = 0.08 * np.hypot(x0[p + n_wall] - x0[p - n_wall], y0[p + n_wall] - y0[p - n_wall]) * 0.5
        jit[p] = rng.uniform(-h, h, 2)
        for dj in (-2, -1, 0, 1, 2):
            for di in (-2, -1, 0, 1, 2):
                if max(abs(dj), abs(di)) < 2:
                    continue
                jj, ii = j + dj, (i + di) % n_wall
                if 0 <= jj < n_radial and rng.random() < 0.35:
                    extra[p].append(jj * n_wall + ii)

    def build():
        x, y = x0 + jit[:, 0], y0 + jit[:, 1]
        lists = [list(nb[p]) + extra[p] for p in range(n)]
        off = np.zeros(n + 1, np.int32)
        off[1:] = np.cumsum([len(l) for l in lists])
        ids = np.array([q for l in lists for q in l], np.int32)
        return x, y, off, ids

    # undo the perturbation around any interior point whose stencil became
    # singular (the reference refuses such clouds, driver.cpp:198-201)
    for _ in range(20):
        x, y, off, ids = build()
        cc = kf.PointCloud.from_arrays(x, y, kind, c.normal_x, c.normal_y, off, ids)
        bad = [p for p in kf.build_ls_coefficients(cc).flagged if kind[p] == 1]

        if not bad:
            break
        for p in bad:
            for q in [p] + list(nb[p]):
                jit[q] = 0.0
                extra[q] = []
    return x, y, kind, c.normal_x.copy(), c.normal_y.copy(), off, ids


def main():
    x, y, kind, nx, ny, off, ids = irregular_cloud()
    ref = Reference.from_arrays(x, y, kind, nx, ny, off, ids)
    out = dict(x=x, y=y, kind=kind, nx=nx, ny=ny, off=off, ids=ids, n_colors=np.array(ref.colors().max()))
    for v in ["explicit", "anandh", "anandh_ad", "manish", "manish_ad"]:
        r = ref.run(variant=v, n_iterations=40, mach=0.63, aoa_deg=2.0, cfl=0.05 if v == "explicit" else 0.2)
        out[v + "_residual"] = r.residual
        out[v + "_cl"] = r.cl
        out[v + "_cd"] = r.cd
        out[v + "_first_order"] = r.first_order
        out[v + "_final"] = r.final_state
        out[v + "_reason"] = np.array(r.abort_reason)
        print(v, len(r.residual), repr(r.abort_reason), int(r.first_order.sum()))
    print("degrees", np.diff(off).min(), np.diff(off).max(), "colours", int(out["n_colors"]))
    np.savez_compressed(os.path.join(HERE, "irregular_histories.npz"), **out)


if __name__ == "__main__":
    main()
