"""The benchmarked BASELINE configurations themselves against the real
reference (oracle/_ref, run on the host in the same test): config 2
(640,000 points, M 0.85, manish_ad: 21 recorded iterations, then an abort)
and config 3 (2,457,600 points, M 1.2, anandh_ad: 6 iterations, then an
abort) -- the same histories to 1e-10, CL/CD, first-order counts and abort
records."""
import os
import sys

import numpy as np
import pytest

import paper_2406_07441_b200 as kf
from util import relmax

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import refpy  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not refpy.ref_available(), reason="reference not built")]

CONFIGS = {
    2: dict(cloud=(1280, 500, 20.0), variant="manish_ad", mach=0.85, aoa=1.0),
    3: dict(cloud=(2560, 960, 20.0), variant="anandh_ad", mach=1.2, aoa=0.0),
}


@pytest.mark.parametrize("config", sorted(CONFIGS))
def test_baseline_config_vs_reference(config):
    c = CONFIGS[config]
    nw, nr, rf = c["cloud"]
    refpy.Reference.num_threads(os.cpu_count() or 1)
    ref = refpy.Reference.generate("0012", nw, nr, rf).run(variant=c["variant"], n_iterations=40, mach=c["mach"],
                                                           aoa_deg=c["aoa"], cfl=0.2)
    cloud = kf.generate_naca_ogrid("0012", nw, nr, rf)
    r = kf.Solver(cloud, kf.SolverConfig(variant=kf.SolverVariant.parse(c["variant"]), mach_inf=c["mach"],
                                         aoa_deg=c["aoa"], cfl=0.2, n_iterations=40)).run()
    assert len(r.iters) == len(ref.residual) and len(r.iters) < 40  # both abort
    assert r.abort_reason == ref.abort_reason
    assert relmax(r.residual, ref.residual) <= 1e-10
    assert np.max(np.abs(r.cl - ref.cl)) <= 1e-10 and np.max(np.abs(r.cd - ref.cd)) <= 1e-10
    assert np.array_equal(r.first_order, ref.first_order)
