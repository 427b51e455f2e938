"""Test helpers (comparisons and cloud plumbing)."""
import numpy as np

import paper_2406_07441_b200 as kf
from refpy import Oracle


def oracle_for(cloud: "kf.PointCloud") -> Oracle:
    """C restatement over exactly the product's ingested arrays."""
    nb = cloud.nbr
    return Oracle(cloud.x, cloud.y, cloud.kind, cloud.normal_x, cloud.normal_y, nb.offsets, nb.ids)


def normrel(a, b):
    """||a - b||_inf / ||b||_inf (R carries cancellation)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.max(np.abs(b)) if b.size else 0.0
    num = np.max(np.abs(a - b)) if b.size else 0.0
    return num / den if den > 0 else num


def relmax(a, b, floor=1e-300):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor))) if b.size else 0.0


def hand_cloud(points, nbrs, kinds=None, normals=None):
    n = len(points)
    x = np.array([p[0] for p in points], np.float64)
    y = np.array([p[1] for p in points], np.float64)
    kind = np.ones(n, np.int32) if kinds is None else np.asarray(kinds, np.int32)
    nx = np.zeros(n)
    ny = np.zeros(n)
    if normals is not None:
        for p, (a, b) in normals.items():
            nx[p], ny[p] = a, b
    off = np.zeros(n + 1, np.int32)
    for p, nb in enumerate(nbrs):
        off[p + 1] = off[p] + len(nb)
    idx = np.array([q for nb in nbrs for q in nb], np.int32)
    return x, y, kind, nx, ny, off, idx


def lattice(nx_, ny_, h=0.1, x0=0.0, y0=0.0):
    pts, nbrs = [], []
    for j in range(ny_):
        for i in range(nx_):
            pts.append((x0 + h * i, y0 + h * j))
    for j in range(ny_):
        for i in range(nx_):
            nb = []
            for dj in (-1, 0, 1):
                for di in (-1, 0, 1):
                    if di == 0 and dj == 0:
                        continue
                    ii, jj = i + di, j + dj
                    if 0 <= ii < nx_ and 0 <= jj < ny_:
                        nb.append(jj * nx_ + ii)
            nbrs.append(nb)
    return pts, nbrs


def shuffled_cloud(c, seed=7):
    """The same cloud under a random point numbering (wall points keep their
    surface-ordered ids, so compute_forces' loop check holds); split stencils,
    LS weights and the greedy colouring are rebuilt by the library."""
    n = c.n()
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
