"""Drop-in edge semantics (round-1 advisor findings):

* n_inner < 1 is not a precondition of run_fixed_point: q_derivatives throws
  inside iteration 1's try block (spatial.cpp:154, driver.cpp:255-262), so
  the run returns diverged, the reason text, no record and the initial state;
* the iteration limit of the device abort key is refused up front;
* step_host validates the caller's arrays before native code sees them.
"""
import os
import sys

import numpy as np
import pytest

import paper_2406_07441_b200 as kf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import refpy  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_parts", [1, 2])
def test_n_inner_zero_aborts_in_iteration_one_like_the_reference(n_parts):
    c = kf.generate_naca_ogrid("0012", 48, 12, 12.0)
    cfg = kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2, n_iterations=5,
                          n_inner=0)
    h = kf.Solver(c, cfg, n_parts=n_parts).run(want_state=True)
    assert h.diverged and h.abort_reason == "q_derivatives: n_inner must be >= 1" and len(h.iters) == 0
    if refpy.ref_available():
        r = refpy.Reference.generate("0012", 48, 12, 12.0).run(variant="manish_ad", n_iterations=5, mach=0.63,
                                                               aoa_deg=2.0, cfl=0.2, n_inner=0)
        assert r.diverged and r.abort_reason == h.abort_reason and len(r.residual) == 0
        assert np.array_equal(h.final_state, r.final_state)
    else:
        # the initial state: free stream + BCs (driver.cpp:207-208)
        s = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0,
                                         n_iterations=1))
        s.reset()
        assert np.array_equal(h.final_state, s.get_state())


def test_step_entry_points_report_the_n_inner_abort():
    c = kf.generate_naca_ogrid("0012", 48, 12, 12.0)
    s = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, n_iterations=5,
                                     n_inner=0))
    U = np.tile(np.array([1.0, 0.6, 0.02, 2.0]), (c.n(), 1))
    with pytest.raises(kf.KinfreeError, match="n_inner"):
        s.step_host(U, np.zeros_like(U))


def test_iteration_limit_is_refused_up_front():
    c = kf.generate_naca_ogrid("0012", 48, 12, 12.0)
    with pytest.raises(kf.ConfigError, match="n_iterations must be <"):
        kf.Solver(c, kf.SolverConfig(n_iterations=(1 << 24)))


def test_step_host_rejects_bad_buffers():
    c = kf.generate_naca_ogrid("0012", 48, 12, 12.0)
    s = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, n_iterations=5))
    s.reset()
    U, dU = s.get_state(with_dU=True)
    with pytest.raises(kf.ConfigError):
        s.step_host(U, None)
    with pytest.raises(kf.ConfigError):
        s.step_host(U[:-1], dU)
    with pytest.raises(kf.ConfigError):
        s.step_host(U, dU, U_out=np.zeros((c.n(), 4), np.float32))
    with pytest.raises(kf.ConfigError):
        s.step_host(U, dU, U_out=np.zeros((c.n(), 8))[:, ::2])
    out, rec = s.step_host(U.astype(np.float32).astype(np.float64), dU)  # converted inputs are fine
    assert out.shape == (c.n(), 4) and np.isfinite(rec.residual)


def test_colour_limit_is_refused_at_create():
    """The device sweeps take at most 120 colours (the abort key's 8-bit
    stage field); a cloud whose greedy colouring needs more -- here a
    121-point clique (far-field boundary points) next to an O-grid -- is refused by kf_create with a
    config error instead of running."""
    base = kf.generate_naca_ogrid("0012", 48, 12, 12.0)
    x, y, kind = list(base.x), list(base.y), list(base.kind)
    nx, ny = list(base.normal_x), list(base.normal_y)
    nb = base.nbr
    lists = [list(nb.ids[nb.offsets[p]:nb.offsets[p + 1]]) for p in range(base.n())]
    m, n0 = 121, base.n()
    rng = np.random.default_rng(5)  # a 2-D blob (no collinear split stencils)
    for k in range(m):
        x.append(30.0 + rng.uniform(-1, 1))
        y.append(30.0 + rng.uniform(-1, 1))
        # (boundary points: a blob's extreme points have one-point split
        # stencils, singular -- refused for interior points, driver.cpp:198-201)
        kind.append(int(kf.PointKind.Outer))
        nx.append(1.0)
        ny.append(0.0)
        lists.append([n0 + j for j in range(m) if j != k])
    off = np.zeros(len(lists) + 1, np.int32)
    np.cumsum([len(a) for a in lists], out=off[1:])
    c = kf.PointCloud.from_arrays(np.array(x), np.array(y), np.array(kind, np.int32), np.array(nx), np.array(ny),
                                  off, np.concatenate(lists).astype(np.int32))
    assert kf.color_points(c).n_colors > 120
    with pytest.raises(kf.ConfigError, match="at most 120"):
        kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, n_iterations=2))
