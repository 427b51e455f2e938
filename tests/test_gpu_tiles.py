"""The SMEM-staged tiles of the gradient and flux kernels do not change any
point's arithmetic: tile formation (breadth-first or plain Morton chunks),
the staged-record cap and the resulting halo batches only move data. States
are therefore BITWISE those of the default tiling; the residual norm, a sum
of per-tile partials, agrees to rounding."""
import os

import numpy as np
import pytest

import paper_2406_07441_b200 as kf
from util import relmax

pytestmark = pytest.mark.gpu


def _run(cloud, env, **kw):
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        base = dict(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2, n_iterations=25)
        base.update(kw)
        s = kf.Solver(cloud, kf.SolverConfig(**base))
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return s.run()


@pytest.mark.parametrize("env", [{"KF_TILE_CAP": "96"}, {"KF_TILE_CAP": "200"}, {"KF_TILE_ORDER": "morton"},
                                 {"KF_GATHER": "ell"}])
@pytest.mark.parametrize("which", ["naca", "irregular"])
def test_tiling_does_not_change_states(env, which):
    if which == "naca":
        c = kf.generate_naca_ogrid("0012", 160, 40, 15.0)
    else:
        g = np.load(os.path.join(os.path.dirname(__file__), "golden", "irregular_histories.npz"))
        c = kf.PointCloud.from_arrays(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["ids"])
    # (the global-gather path has one thread per point: compare it with the
    # one-thread tile kernel, not the two-thread small-cloud variant)
    base = {"KF_RES_SPLIT_MAX": "0"} if "KF_GATHER" in env else {}
    a = _run(c, base)
    b = _run(c, {**env, **base})
    assert len(a.iters) == len(b.iters) and a.abort_reason == b.abort_reason
    assert np.array_equal(a.final_state, b.final_state)
    assert np.array_equal(a.cl, b.cl) and np.array_equal(a.first_order, b.first_order)
    assert relmax(a.residual, b.residual) <= 1e-13


@pytest.mark.parametrize("variant", ["manish_ad", "anandh"])
def test_two_thread_flux_variant_matches_one_thread(variant):
    """Clouds under KF_RES_SPLIT_MAX points run the flux kernel with two
    threads per point (even / odd stencil entries, one extra addition): the
    same demotions, tallies and abort record, states equal to rounding."""
    c = kf.generate_naca_ogrid("0012", 160, 40, 15.0)
    a = _run(c, {"KF_RES_SPLIT_MAX": "0"}, variant=kf.SolverVariant.parse(variant))
    b = _run(c, {"KF_RES_SPLIT_MAX": "100000000"}, variant=kf.SolverVariant.parse(variant))
    assert len(a.iters) == len(b.iters) and a.abort_reason == b.abort_reason
    assert np.array_equal(a.first_order, b.first_order)
    assert np.array_equal(np.array([i.counters for i in a.iters]), np.array([i.counters for i in b.iters]))
    assert relmax(a.residual, b.residual) <= 1e-12
    d = np.abs(a.final_state - b.final_state).max() / np.abs(a.final_state).max()
    assert d <= 1e-12


def test_hub_point_cloud_falls_back_to_global_gathers():
    """A cloud with a hub point of 700 neighbours (wider than a tile's shared
    memory can stage) runs the global-gather kernels automatically and keeps
    the reference's history."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import refpy
    if not refpy.ref_available():
        pytest.skip("reference library not built")
    base = kf.generate_naca_ogrid("0012", 96, 24, 12.0)
    x, y, kind = base.x.copy(), base.y.copy(), base.kind.copy()
    nx, ny = base.normal_x.copy(), base.normal_y.copy()
    off, ids = base.nbr.offsets.copy(), base.nbr.ids.copy()
    inner = np.flatnonzero(kind == kf.PointKind.Interior)
    p = inner[len(inner) // 2]
    hx, hy = x[p] + 1e-3, y[p] + 1e-3
    d = np.hypot(x - hx, y - hy)
    hub_nb = np.argsort(d)[:700]
    x, y = np.append(x, hx), np.append(y, hy)
    kind = np.append(kind, int(kf.PointKind.Interior))
    nx, ny = np.append(nx, 0.0), np.append(ny, 0.0)
    ids = np.concatenate([ids, hub_nb]).astype(np.int32)
    off = np.append(off, off[-1] + len(hub_nb)).astype(np.int32)
    c = kf.PointCloud.from_arrays(x, y, kind, nx, ny, off, ids)
    cfg = kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2, n_iterations=20)
    r = kf.Solver(c, cfg).run()
    ref = refpy.Reference.from_arrays(x, y, kind, nx, ny, off, ids).run(variant="manish_ad", n_iterations=20,
                                                                         mach=0.63, aoa_deg=2.0, cfl=0.2)
    # (so wide a stencil makes the hub's residual overflow at once: both stop
    # on the same record with the same abort; compare the finite entries)
    assert len(r.iters) == len(ref.residual) and r.abort_reason == ref.abort_reason
    fin = np.isfinite(ref.residual)
    assert np.array_equal(np.isfinite(r.residual), fin)
    assert relmax(r.residual[fin], ref.residual[fin]) <= 1e-10
    assert np.max(np.abs(r.cl - ref.cl)) <= 1e-10
