"""The domain-decomposed solver on one B200.

Partitions are held in-process on one device (ghosts refreshed by device
copies between dependent stages, residual/forces/abort keys reduced across
partitions every iteration). The multi-process NCCL transport runs the same
kernels, layouts and exchange schedule; only the copy calls differ.

Expectations:
  * per-point arithmetic is the single-partition arithmetic on bitwise-equal
    inputs (ghosts are exact copies, colours are global), so states after
    every iteration are BITWISE equal to the unpartitioned run;
  * only the residual sum is reassociated (per-partition partials), so the
    residual history matches to <= 1e-13 relative and CL/CD exactly;
  * against the reference the usual 1e-10 run contract holds, including the
    config-1 abort record.
"""
import os

import numpy as np
import pytest

import paper_2406_07441_b200 as kf
from util import normrel, relmax

pytestmark = pytest.mark.gpu

VARIANTS = ["explicit", "anandh", "anandh_ad", "manish", "manish_ad"]


@pytest.fixture(scope="module")
def small():
    return kf.generate_naca_ogrid("0012", 48, 12, 12.0)


def cfg(variant, **kw):
    base = dict(variant=kf.SolverVariant.parse(variant), mach_inf=0.63, aoa_deg=2.0,
                cfl=0.05 if variant == "explicit" else 0.2)
    base.update(kw)
    return kf.SolverConfig(**base)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("n_parts,mode", [(2, "angular"), (3, "morton"), (5, "angular")])
def test_partitioned_history_matches_single_and_reference(golden, small, variant, n_parts, mode):
    h = np.load(os.path.join(golden, "small_histories.npz"))
    one = kf.Solver(small, cfg(variant, n_iterations=60)).run()
    s = kf.Solver(small, cfg(variant, n_iterations=60), n_parts=n_parts, partition=mode)
    assert s.n_parts == n_parts and s.owned_points == small.n()
    r = s.run()
    assert len(r.iters) == len(one.iters)
    assert r.abort_reason == one.abort_reason
    assert relmax(r.residual, one.residual) <= 1e-13
    assert np.array_equal(r.cl, one.cl) and np.array_equal(r.cd, one.cd)
    assert np.array_equal(r.final_state, one.final_state)
    assert np.array_equal(np.array([i.counters for i in r.iters]), np.array([i.counters for i in one.iters]))
    assert np.array_equal(r.first_order, one.first_order)
    # and the reference contract
    assert relmax(r.residual, h[variant + "_residual"]) <= 1e-10
    assert np.max(np.abs(r.cl - h[variant + "_cl"])) <= 1e-10


@pytest.mark.parametrize("n_inner", [1, 2, 4, 5])
def test_partitioned_n_inner_is_bitwise_single(small, n_inner):
    """Every gradient-pass count, partitioned vs single: the last pass of an
    even count leaves the flux kernel's q in buffer 1 (carried there by that
    pass, ghosts by the halo exchange), an odd count in buffer 0."""
    one = kf.Solver(small, cfg("manish_ad", n_iterations=12, n_inner=n_inner)).run()
    r = kf.Solver(small, cfg("manish_ad", n_iterations=12, n_inner=n_inner), n_parts=3).run()
    assert len(r.iters) == len(one.iters) == 12, (r.abort_reason, one.abort_reason)
    assert np.array_equal(r.final_state, one.final_state)
    assert np.array_equal(r.cl, one.cl) and relmax(r.residual, one.residual) <= 1e-13


def test_partitioned_state_is_bitwise_single_every_iteration(small):
    a = kf.Solver(small, cfg("manish_ad", n_iterations=20))
    b = kf.Solver(small, cfg("manish_ad", n_iterations=20), n_parts=4)
    a.reset()
    b.reset()
    for _ in range(6):
        a.iterate_async(1)
        b.iterate_async(1)
        Ua, dUa = a.get_state(with_dU=True)
        Ub, dUb = b.get_state(with_dU=True)
        assert np.array_equal(Ua, Ub) and np.array_equal(dUa, dUb)


def test_partitioned_config1_trajectory_and_abort(golden):
    """Config 1 (38,400 points) split in 4 wedges: the reference's 422
    recorded iterations and its abort record in iteration 423."""
    h = np.load(os.path.join(golden, "config1_history.npz"))
    c = kf.generate_naca_ogrid("0012", 320, 120, 20.0)
    s = kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD, mach_inf=0.63, aoa_deg=2.0,
                                     cfl=0.2, n_iterations=1000), n_parts=4)
    r = s.run()
    assert len(r.iters) == 422
    assert r.diverged and r.abort_reason == "nonpositive density at point 27005"
    assert r.abort_point == 27005
    assert relmax(r.residual, h["residual"]) <= 1e-10
    assert np.max(np.abs(r.cl - h["cl"])) <= 1e-10 and np.max(np.abs(r.cd - h["cd"])) <= 1e-10
    assert np.array_equal(r.first_order, h["first_order"])


def test_partitioned_bench_and_step_host(small):
    one = kf.Solver(small, cfg("manish_ad", n_iterations=16))
    par = kf.Solver(small, cfg("manish_ad", n_iterations=16), n_parts=3, partition="morton")
    for s in (one, par):
        s.reset()
        s.iterate_async(4)
        s.sync_records()
    U0, dU0 = one.get_state(with_dU=True)
    Ua, ra = one.step_host(U0, dU0)
    Ub, rb = par.step_host(U0, dU0)
    assert np.array_equal(Ua, Ub)
    assert abs(ra.residual - rb.residual) <= 1e-13 * abs(ra.residual) and ra.cl == rb.cl
    # bench mode: every step re-runs the same iteration from the snapshot
    par.set_state(U0, dU0)
    par.bench_mode(True)
    par.iterate_async(3)
    recs, st = par.sync_records()
    assert st.code == 0
    assert abs(recs[0].residual - ra.residual) <= 1e-13 * abs(ra.residual)
    assert par.launches_per_iteration > one.launches_per_iteration


def test_partitioned_contexts_refuse_stage_hooks(small):
    s = kf.Solver(small, cfg("manish_ad"), n_parts=2)
    with pytest.raises(kf.ConfigError):
        s.q(np.ones((small.n(), 4)))


def test_nccl_transport_single_rank(small):
    """The NCCL transport with one rank (the path every rank of a multi-GPU
    run takes: NCCL bound at run time, communicator, halo groups and the
    per-iteration ncclAllReduce captured in the iteration graph, reduced
    records through k_finalize<MULTI>) against the unpartitioned solver."""
    one = kf.Solver(small, cfg("manish_ad", n_iterations=40)).run()
    s = kf.Solver.for_rank(small, cfg("manish_ad", n_iterations=40), 1, 0, kf.nccl_unique_id())
    assert s.n_parts == 1 and s.owned_points == small.n()
    r = s.run()
    assert len(r.iters) == len(one.iters) and r.abort_reason == one.abort_reason
    assert relmax(r.residual, one.residual) <= 1e-13
    assert np.array_equal(r.cl, one.cl)
    assert np.array_equal(r.final_state, one.final_state)
    # stepping and the host-fed step through the same transport
    s.reset()
    s.iterate_async(3)
    U, dU = s.get_state(with_dU=True)
    got, rec = s.step_host(U, dU)
    ref = kf.Solver(small, cfg("manish_ad", n_iterations=40))
    want, rec1 = ref.step_host(U, dU)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("use_graph", [True, False])
def test_many_partitions_and_eager_launches(small, use_graph):
    """12 Morton partitions of a 576-point cloud (partitions with empty colour
    blocks, many peers) and the eager (non-graph) launch path: states bitwise
    the unpartitioned graph run."""
    one = kf.Solver(small, cfg("anandh", n_iterations=25)).run()
    r = kf.Solver(small, cfg("anandh", n_iterations=25, use_graph=use_graph), n_parts=12,
                  partition="morton").run()
    assert len(r.iters) == len(one.iters) and r.abort_reason == one.abort_reason
    assert np.array_equal(r.final_state, one.final_state)
    assert relmax(r.residual, one.residual) <= 1e-13 and np.array_equal(r.cl, one.cl)


@pytest.mark.parametrize("variant", ["manish_ad", "anandh", "explicit"])
@pytest.mark.parametrize("n_parts,mode,nw,nr", [(4, "angular", 320, 120), (3, "morton", 96, 33)])
def test_overlapped_exchanges_are_bitwise_single(monkeypatch, variant, n_parts, mode, nw, nr):
    """KF_OVERLAP=1: every gradient pass and sweep colour runs its boundary
    tiles / points first, exchanges their halo on a second stream while the
    interior runs, and joins before the next stage (the NCCL transport's
    default). States, histories and the abort record stay bitwise those of
    the unpartitioned run."""
    c = kf.generate_naca_ogrid("0012", nw, nr, 20.0)
    one = kf.Solver(c, cfg(variant, n_iterations=40)).run(want_state=True)
    monkeypatch.setenv("KF_OVERLAP", "1")
    r = kf.Solver(c, cfg(variant, n_iterations=40), n_parts=n_parts, partition=mode).run(want_state=True)
    assert len(r.iters) == len(one.iters) and r.abort_reason == one.abort_reason
    assert np.array_equal(r.final_state, one.final_state)
    assert np.array_equal(r.cl, one.cl) and relmax(r.residual, one.residual) <= 1e-13
