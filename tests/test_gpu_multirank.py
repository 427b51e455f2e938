"""Multi-process decomposition on the GPU: one process per rank, halos and
the per-iteration reduction moved by a real inter-process communicator
(torch.distributed gloo over 127.0.0.1) through the host-staged transport
(kf_create_rank_host). Every rank runs the rank-local setup, compact I/O,
posted message list and reduced records of the multi-GPU path; only the wire
differs from NCCL (the NCCL transport itself is exercised with one rank in
test_gpu_partition.py, and NCCL refuses two ranks on one device).

Expectations as for the in-process partitions: each rank's owned states are
BITWISE the unpartitioned run's, CL/CD bitwise, the residual within 1e-13
(reassociated sum), and config 1 reproduces the reference's 422 iterations
and abort record on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2406_07441_b200 as kf
from util import relmax

pytestmark = pytest.mark.gpu

CASES = {
    "small_manish_ad": dict(cloud=("0012", 48, 12, 12.0), variant="manish_ad", iters=60, world=2, mode="angular"),
    "small_anandh_morton": dict(cloud=("0012", 48, 12, 12.0), variant="anandh", iters=40, world=3, mode="morton"),
    "config1": dict(cloud=("0012", 320, 120, 20.0), variant="manish_ad", iters=1000, world=4, mode="angular"),
}


def _cfg(variant, iters):
    return kf.SolverConfig(variant=kf.SolverVariant.parse(variant), mach_inf=0.63, aoa_deg=2.0,
                           cfl=0.05 if variant == "explicit" else 0.2, n_iterations=iters)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        case = CASES[name]
        c = kf.generate_naca_ogrid(*case["cloud"])

        def exchange(msgs):
            reqs = []
            for peer, is_send, buf in msgs:
                t = torch.from_numpy(buf)
                reqs.append(dist.isend(t, peer) if is_send else dist.irecv(t, peer))
            for r in reqs:
                r.wait()

        def allreduce(buf):
            dist.all_reduce(torch.from_numpy(buf))

        s = kf.Solver.for_rank_host(c, _cfg(case["variant"], case["iters"]), world, rank, exchange, allreduce,
                                    partition=case["mode"])
        assert s.n_parts == world
        r = s.run()
        # the C-ABI host step on this rank (only its own points are read and
        # written: the host arrays keep the whole-cloud shape)
        s.reset()
        s.iterate_async(3)
        U, dU = s.get_state(with_dU=True)
        Us, rec = s.step_host(U, dU)
        q.put((rank, None, r.residual, r.cl, r.cd, r.abort_reason, r.final_state, s.owned_points, Us,
               rec.residual))
        s.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc() + repr(e), None, None, None, None, None, None, None, None))


@pytest.mark.parametrize("name", sorted(CASES))
def test_ranks_over_host_communicator_match_single(name):
    case = CASES[name]
    world = case["world"]
    c = kf.generate_naca_ogrid(*case["cloud"])
    single = kf.Solver(c, _cfg(case["variant"], case["iters"]))
    one = single.run()
    single.reset()
    single.iterate_async(3)
    U3, dU3 = single.get_state(with_dU=True)
    one_step, one_rec = single.step_host(U3, dU3)
    owner = kf.partition_plan(c, world, case["mode"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    owned_total = 0
    for rank, err, residual, cl, cd, reason, state, n_owned, step_state, step_res in sorted(res, key=lambda x: x[0]):
        assert err is None, err
        assert len(residual) == len(one.iters) and reason == one.abort_reason
        assert relmax(residual, one.residual) <= 1e-13
        assert np.array_equal(cl, one.cl) and np.array_equal(cd, one.cd)
        mine = owner == rank
        assert n_owned == int(mine.sum())
        assert np.array_equal(state[mine], one.final_state[mine])
        if len(one.iters) > 3:
            assert np.array_equal(step_state[mine], one_step[mine])
            assert abs(step_res - one_rec.residual) <= 1e-13 * abs(one_rec.residual)
        owned_total += n_owned
    assert owned_total == c.n()
    if name == "config1":
        assert len(one.iters) == 422 and one.abort_reason == "nonpositive density at point 27005"
