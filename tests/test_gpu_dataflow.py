"""Dataflow LU-SGS sweeps (kernels.cuh k_forward_df / k_backward_df; the
default from 4M points, KF_SWEEP_DF=1 forces them on any single-partition
cloud): one launch per sweep direction, 32-point slices handed out in a
level-skewed topological order, each slice waiting on the release flags of
the slices its gathers read. Only the schedule changes -- every point runs
the per-colour kernels' arithmetic on the same inputs -- so states, histories,
tallies and abort records are BITWISE those of the per-colour launches
(implicit.cpp:153-226 order of evaluation per point)."""
import os

import numpy as np
import pytest

import paper_2406_07441_b200 as kf

pytestmark = pytest.mark.gpu


def _run(cloud, df, want_state=True, **kw):
    saved = os.environ.get("KF_SWEEP_DF")
    os.environ["KF_SWEEP_DF"] = "1" if df else "0"
    try:
        base = dict(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0, cfl=0.2, n_iterations=30)
        base.update(kw)
        s = kf.Solver(cloud, kf.SolverConfig(**base))
    finally:
        if saved is None:
            os.environ.pop("KF_SWEEP_DF", None)
        else:
            os.environ["KF_SWEEP_DF"] = saved
    return s.run(want_state=want_state)


def _same(a, b):
    assert len(a.iters) == len(b.iters) and a.abort_reason == b.abort_reason
    assert a.diverged == b.diverged
    assert np.array_equal(a.final_state, b.final_state)
    assert np.array_equal(a.residual, b.residual)
    assert np.array_equal(a.cl, b.cl) and np.array_equal(a.cd, b.cd)
    assert np.array_equal(a.first_order, b.first_order)
    assert np.array_equal(np.array([i.counters for i in a.iters]), np.array([i.counters for i in b.iters]))


def _irregular():
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "irregular_histories.npz"))
    return kf.PointCloud.from_arrays(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["ids"])


@pytest.mark.parametrize("variant", ["anandh", "anandh_ad", "manish", "manish_ad"])
@pytest.mark.parametrize("which", ["naca", "irregular"])
def test_dataflow_sweeps_bitwise_per_colour(variant, which):
    c = kf.generate_naca_ogrid("0012", 160, 40, 15.0) if which == "naca" else _irregular()
    kw = dict(variant=kf.SolverVariant.parse(variant), n_iterations=40)
    _same(_run(c, True, **kw), _run(c, False, **kw))


@pytest.mark.parametrize("plan", ["jp_hash", "wall_first"])
def test_dataflow_sweeps_other_colourings(plan):
    """More colours (device Jones-Plassmann on a hashed priority; the paper's
    wall-first levels): longer dependency chains, same results."""
    c = kf.generate_naca_ogrid("0012", 192, 48, 15.0)
    if plan == "jp_hash":
        kf.color_points_device(c, "hash", seed=3)
    else:
        kf.order_wall_first(c)
    _same(_run(c, True, n_iterations=30), _run(c, False, n_iterations=30))


def test_dataflow_sweeps_config1_abort_record():
    """Config 1 to its abort (422 records, the abort in iteration 423 at
    point 27005, the reference's record): the epoch-flagged schedule over
    hundreds of graph-launched iterations."""
    c = kf.generate_naca_ogrid("0012", 320, 120, 20.0)
    a = _run(c, True, n_iterations=430)
    b = _run(c, False, n_iterations=430)
    _same(a, b)
    assert a.diverged and len(a.iters) == 422
    assert a.abort_reason == "nonpositive density at point 27005"


def test_dataflow_sweeps_host_steps():
    """The host-fed step (kf_step_host, the e2e path) on the dataflow
    schedule: bitwise the per-colour step."""
    c = kf.generate_naca_ogrid("0012", 160, 40, 15.0)
    outs = []
    for df in (True, False):
        os.environ["KF_SWEEP_DF"] = "1" if df else "0"
        try:
            s = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0,
                                             cfl=0.2, n_iterations=3))
        finally:
            os.environ.pop("KF_SWEEP_DF", None)
        s.run()
        U, dU = s.get_state(with_dU=True)
        for _ in range(5):
            U2, dU2 = np.zeros_like(U), np.zeros_like(U)
            s.step_host(U, dU, U_out=U2, dU_out=dU2)
            U, dU = U2, dU2
        outs.append((U, dU))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
