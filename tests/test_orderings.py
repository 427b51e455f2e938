"""Sweep-ordering variants, host side: the paper's
Algorithm 5 wall-first levels built from a colouring.
The device colouring and the solver runs are in tests/test_gpu_orderings.py."""
import numpy as np

import paper_2406_07441_b200 as kf


def _sym_edges(c):
    n = c.n()
    src = np.repeat(np.arange(n), np.diff(c.nbr.offsets))
    a, b = np.concatenate([src, c.nbr.ids]), np.concatenate([c.nbr.ids, src])
    m = a != b
    return a[m], b[m]


def test_wall_first_levels_are_a_valid_kind_major_order():
    # odd n_radial: the outer ring gets low greedy colours, so the levels
    # really reorder it behind the interior
    c = kf.generate_naca_ogrid("0012", 64, 17, 12.0)
    old = kf.color_points(c).color.copy()
    lev = kf.order_wall_first(c)
    L = lev.color
    a, b = _sym_edges(c)
    assert not np.any(L[a] == L[b])  # still a colouring
    assert set(np.unique(L)) == set(range(1, lev.n_colors + 1))  # no empty level
    rank = np.where(c.kind == 0, 0, np.where(c.kind == 1, 1, 2))
    # kind-major: every wall level precedes every interior level precedes every outer level
    for k0, k1 in [(0, 1), (1, 2)]:
        assert L[rank == k0].max() < L[rank == k1].min()
    # inside a kind the greedy colour order is kept
    for k in range(3):
        m = rank == k
        o, l = old[m], L[m]
        assert np.all(np.diff(l[np.argsort(o, kind="stable")]) >= 0)
    # the outer ring moved: some outer point was below some interior point before
    assert np.any(old[rank == 2].min() < old[rank == 1].max())
    # the library adopted it (the solver sweeps these levels)
    assert np.array_equal(kf.color_points(c).color, L)
