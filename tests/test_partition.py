"""Host logic of the domain decomposition, on CPU.

The planner and local layouts are pure host C++ (partition.cpp, exposed
through kf_partition_plan / kf_layout_*). These tests check the invariants the
device path relies on, and replay the exact per-iteration message pattern of
the NCCL transport (per peer, per colour: send list -> ghost range, in the
same order) over a world-size-2 gloo process group.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2406_07441_b200 as kf


@pytest.fixture(scope="module")
def cloud():
    return kf.generate_naca_ogrid("0012", 64, 20, 12.0)


def _bc_sources(c):
    """nearest_interior_neighbour (driver.cpp:51-65): first minimum in nbr order."""
    nb = c.nbr
    src = np.full(c.n(), -1)
    for p in range(c.n()):
        best = np.inf
        for i in nb[p]:
            d = np.hypot(c.x[i] - c.x[p], c.y[i] - c.y[p])
            if c.kind[i] == kf.PointKind.Interior and d < best:
                best, src[p] = d, i
    return src


@pytest.mark.parametrize("mode", ["angular", "morton"])
@pytest.mark.parametrize("n_parts", [1, 2, 3, 8])
def test_plan_balanced_and_keeps_bc_sources_local(cloud, n_parts, mode):
    owner = kf.partition_plan(cloud, n_parts, mode)
    assert owner.shape == (cloud.n(),) and owner.min() >= 0 and owner.max() == n_parts - 1
    counts = np.bincount(owner, minlength=n_parts)
    # equal-count chunks, then outer points follow their BC source
    assert counts.max() - counts.min() <= 0.1 * cloud.n() / n_parts + 64
    src = _bc_sources(cloud)
    outer = np.flatnonzero(cloud.kind == kf.PointKind.Outer)
    ok = src[outer] >= 0
    assert np.array_equal(owner[outer[ok]], owner[src[outer[ok]]])


def test_plan_rejects_bad_arguments(cloud):
    with pytest.raises(kf.KinfreeError):
        kf.partition_plan(cloud, 0)
    with pytest.raises(ValueError):
        kf.partition_plan(cloud, 2, "spiral")


@pytest.mark.parametrize("mode", ["angular", "morton"])
@pytest.mark.parametrize("n_parts", [2, 4, 7])
def test_layouts_are_consistent_across_ranks(cloud, n_parts, mode):
    owner = kf.partition_plan(cloud, n_parts, mode)
    colors = kf.color_points(cloud).color
    nb = cloud.nbr
    Ls = [kf.LocalLayout(cloud, owner, n_parts, r) for r in range(n_parts)]
    assert sum(L.n_owned for L in Ls) == cloud.n()
    for r, L in enumerate(Ls):
        real = L.perm >= 0
        owned = real & (L.ghost == 0)
        # owned set = owner's points; ghosts = non-owned 1-ring neighbours
        assert np.array_equal(np.sort(L.perm[owned]), np.flatnonzero(owner == r))
        want_ghosts = set()
        for p in np.flatnonzero(owner == r):
            want_ghosts.update(int(i) for i in nb[p] if owner[i] != r)
        assert set(L.perm[real & (L.ghost == 1)].tolist()) == want_ghosts
        # colour-major blocks, owned then ghosts, warp padded
        for c in range(L.n_colors):
            assert L.gs[c] % 32 == 0 and L.oe[c] % 32 == 0 and L.ge[c] % 32 == 0
            blk = L.perm[L.gs[c]:L.ge[c]]
            assert np.all(colors[blk[blk >= 0]] == c + 1)
            assert not L.ghost[L.gs[c]:L.oe[c]].any()
            seg = L.ghost[L.oe[c]:L.ge[c]]
            assert np.all(seg[L.perm[L.oe[c]:L.ge[c]] >= 0] == 1)
        assert set(L.peers.tolist()) == {int(owner[g]) for g in want_ghosts} | {
            s for s in range(n_parts) if s != r and any(owner[i] == r for p in np.flatnonzero(owner == s)
                                                        for i in nb[p])}
    # every message: what rank a sends to b in colour c is exactly the ghost
    # range b fills from a in colour c, element by element
    for a, La in enumerate(Ls):
        for ka, b in enumerate(La.peers):
            Lb = Ls[b]
            kb = int(np.flatnonzero(Lb.peers == a)[0])
            for c in range(La.n_colors):
                sent = La.send(ka, c)
                off, cnt = Lb.recv(kb, c)
                assert cnt == len(sent)
                assert np.array_equal(Lb.perm[off:off + cnt], sent)
                assert np.all(owner[sent] == a) and np.all(colors[sent] == c + 1)


@pytest.mark.parametrize("asym", [False, True])
@pytest.mark.parametrize("n_parts", [2, 3])
def test_layout_boundary_first(cloud, n_parts, asym):
    """Inside each colour block the owned points a peer needs or that read a
    ghost come first, [gs, ob); the interior [ob, oe) neither feeds nor reads
    the halo, which is what lets the solver overlap the exchange with it --
    also for asymmetric stencils (extra one-way neighbours)."""
    c = cloud
    if asym:
        rng = np.random.default_rng(3)
        nb = c.nbr
        lists = [list(nb[p]) for p in range(c.n())]
        inner = np.flatnonzero(c.kind == kf.PointKind.Interior)
        for p in rng.choice(inner, 200, replace=False):
            d = np.hypot(c.x - c.x[p], c.y - c.y[p])
            q = int(np.argsort(d)[12])  # a one-way neighbour, two rings out
            if q not in lists[p] and q != p:
                lists[p].append(q)
        off = np.zeros(c.n() + 1, np.int32)
        np.cumsum([len(a) for a in lists], out=off[1:])
        c = kf.PointCloud.from_arrays(c.x, c.y, c.kind.astype(np.int32), c.normal_x, c.normal_y, off,
                                      np.concatenate(lists).astype(np.int32))
    owner = kf.partition_plan(c, n_parts, "angular")
    nb = c.nbr
    for r in range(n_parts):
        L = kf.LocalLayout(c, owner, n_parts, r)
        sent = set()
        for k in range(L.n_peers):
            for cc in range(L.n_colors):
                sent.update(L.send(k, cc).tolist())
        for cc in range(L.n_colors):
            assert L.gs[cc] <= L.ob[cc] <= L.oe[cc]
            for pn in range(L.gs[cc], L.oe[cc]):
                g = int(L.perm[pn])
                if g < 0:
                    continue
                bnd = g in sent or any(owner[i] != r for i in nb[g])
                assert bnd == (pn < L.ob[cc]), (r, cc, pn)


def test_single_partition_layout_has_no_halo(cloud):
    L = kf.LocalLayout(cloud, np.zeros(cloud.n(), np.int32), 1, 0)
    assert L.n_peers == 0 and not L.ghost.any() and np.array_equal(L.oe, L.ge)
    assert L.n_owned == cloud.n()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange_worker(rank, world, port, q):
    """One rank of the halo exchange, message for message as the NCCL
    transport issues it (exchange_rec: per peer, per colour, send the
    packed records, receive into the ghost range)."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        c = kf.generate_naca_ogrid("0012", 64, 20, 12.0)
        owner = kf.partition_plan(c, world, "angular")
        L = kf.LocalLayout(c, owner, world, rank)
        # a per-point payload with a known value per global point: (gid, x, y)
        buf = np.full((L.n_local, 3), -1.0)
        own = (L.perm >= 0) & (L.ghost == 0)
        buf[own] = np.stack([L.perm[own], c.x[L.perm[own]], c.y[L.perm[own]]], 1)
        inv = {int(g): k for k, g in enumerate(L.perm) if g >= 0}
        reqs, recvs = [], []
        for k, peer in enumerate(L.peers):
            for col in range(L.n_colors):
                sent = L.send(k, col)
                if len(sent):
                    pkt = torch.from_numpy(np.ascontiguousarray(buf[[inv[int(g)] for g in sent]]))
                    reqs.append(dist.isend(pkt, int(peer)))
                off, cnt = L.recv(k, col)
                if cnt:
                    t = torch.empty((cnt, 3), dtype=torch.float64)
                    reqs.append(dist.irecv(t, int(peer)))
                    recvs.append((off, cnt, t))
        for r in reqs:
            r.wait()
        for off, cnt, t in recvs:
            buf[off:off + cnt] = t.numpy()
        ghost = (L.perm >= 0) & (L.ghost == 1)
        g = L.perm[ghost]
        ok = (np.array_equal(buf[ghost, 0], g) and np.array_equal(buf[ghost, 1], c.x[g])
              and np.array_equal(buf[ghost, 2], c.y[g]))
        n_ghost = int(ghost.sum())
        tot = torch.tensor([n_ghost], dtype=torch.int64)
        dist.all_reduce(tot)
        q.put((rank, ok, n_ghost, int(tot.item())))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e), 0))


def test_halo_exchange_pattern_over_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, n_ghost, tot in sorted(res):
        assert ok, (rank, n_ghost)
        assert n_ghost > 0 and tot > n_ghost


def test_rcm_ordering_layout(cloud):
    """ordering 2 (reverse Cuthill-McKee inside each colour block): a
    permutation of the same blocks, with a smaller mean neighbour distance
    in local numbering than the natural order would give on a shuffled cloud
    (here: still a valid colour-major layout with every point once)."""
    L0 = kf.LocalLayout(cloud, np.zeros(cloud.n(), np.int32), 1, 0, ordering=0)
    L2 = kf.LocalLayout(cloud, np.zeros(cloud.n(), np.int32), 1, 0, ordering=2)
    assert np.array_equal(L0.gs, L2.gs) and np.array_equal(L0.oe, L2.oe)
    for c in range(L0.n_colors):
        a = L0.perm[L0.gs[c]:L0.oe[c]]
        b = L2.perm[L2.gs[c]:L2.oe[c]]
        assert np.array_equal(np.sort(a[a >= 0]), np.sort(b[b >= 0]))
    assert not np.array_equal(L0.perm, L2.perm)
