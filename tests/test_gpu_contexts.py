"""Several solver contexts in one process on one device: each owns its
stream, graphs and buffers, and the process-wide kernel attributes (the
tile kernels' dynamic shared-memory limit) never drop below what another
live context launches with. Interleaved iteration gives every context
exactly its solo results."""
import numpy as np
import pytest

import paper_2406_07441_b200 as kf

pytestmark = pytest.mark.gpu


def _cfg(variant, iters):
    return kf.SolverConfig(variant=kf.SolverVariant.parse(variant), mach_inf=0.63, aoa_deg=2.0,
                           cfl=0.05 if variant == "explicit" else 0.2, n_iterations=iters)


def test_interleaved_contexts_match_solo_runs():
    big = kf.generate_naca_ogrid("0012", 192, 64, 20.0)
    small = kf.generate_naca_ogrid("0012", 48, 12, 12.0)
    specs = [(big, "manish_ad", 1), (small, "anandh", 3), (big, "explicit", 1)]
    solo = []
    for c, v, parts in specs:
        s = kf.Solver(c, _cfg(v, 12), n_parts=parts)
        s.reset()
        s.iterate_async(12)
        recs, _ = s.sync_records()
        solo.append((s.get_state(with_dU=True), [r.residual for r in recs]))
        s.close()
    live = [kf.Solver(c, _cfg(v, 12), n_parts=parts) for c, v, parts in specs]
    for s in live:
        s.reset()
    for _ in range(12):
        for k, s in enumerate(live):  # round-robin, one iteration each
            s.iterate_async(1)
    for k, s in enumerate(live):
        recs, _ = s.sync_records()
        U, dU = s.get_state(with_dU=True)
        assert np.array_equal(U, solo[k][0][0]) and np.array_equal(dU, solo[k][0][1])
        assert [r.residual for r in recs] == solo[k][1]
    for s in live:
        s.close()
