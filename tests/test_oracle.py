"""Pin the checker before trusting it (CPU only).

The plain-C restatement (oracle/kf_oracle.c) must reproduce the reference
bit-for-bit: against the committed golden fixtures produced by the real
reference (tests/golden/make_golden.py), and against the live reference
build (oracle/_ref) where /root/reference exists. Plus the reference test
suite's own known-answer checks on the point physics
(tests/test_kinetics.cpp, tests/test_tangent.cpp).
"""
import json
import os

import numpy as np
import pytest

from refpy import Oracle, Reference, ref_available, oracle_from_reference
from util import hand_cloud, lattice

import paper_2406_07441_b200 as kf

GAMMA = 1.4


def small_oracle():
    c = kf.generate_naca_ogrid("0012", 48, 12, 12.0)
    nb = c.nbr
    return Oracle(c.x, c.y, c.kind, c.normal_x, c.normal_y, nb.offsets, nb.ids)


@pytest.mark.parametrize("variant", ["explicit", "anandh", "anandh_ad", "manish", "manish_ad"])
def test_oracle_stages_bitwise_vs_golden(golden, variant):
    g = np.load(os.path.join(golden, f"stages_{variant}.npz"))
    o = small_oracle()
    U = g["U"]
    q = o.q(U)
    assert np.array_equal(q, g["q"])
    qx, qy = o.grads(q, 3)
    assert np.array_equal(qx, g["qx"]) and np.array_equal(qy, g["qy"])
    R, dem = o.residual(q, qx, qy)
    assert np.array_equal(R, g["R"]) and np.array_equal(dem, g["demoted"])
    cfl = float(g["cfl"])
    dt = o.timestep(U, cfl)
    assert np.array_equal(dt, g["dt"])
    if variant == "explicit":
        return
    exact = variant.endswith("_ad")
    S = None
    if variant.startswith("manish"):
        S, _ = o.s_term(U, g["dU_prev"], exact)
        assert np.array_equal(S, g["S"])
    d = o.diagonal(U, dt, variant)
    assert np.array_equal(d, g["diag"])
    dUs, dU = o.sweeps(U, R, S, d, exact)
    assert np.array_equal(dUs, g["dU_star"]) and np.array_equal(dU, g["dU"])
    Un = o.bc(U + dU, float(g["mach"]), float(g["aoa"]))
    assert np.array_equal(Un, g["U_next"])
    cl, cd = o.forces(Un, float(g["mach"]), float(g["aoa"]))
    assert cl == float(g["cl"]) and cd == float(g["cd"])


def test_oracle_small_histories_bitwise(golden):
    h = np.load(os.path.join(golden, "small_histories.npz"))
    o = small_oracle()
    for v in ["explicit", "anandh", "anandh_ad", "manish", "manish_ad"]:
        cfl = 0.05 if v == "explicit" else 0.2
        r = o.run(variant=v, n_iterations=60, mach=0.63, aoa_deg=2.0, cfl=cfl)
        assert np.array_equal(r.residual, h[v + "_residual"]), v
        assert np.array_equal(r.cl, h[v + "_cl"]) and np.array_equal(r.cd, h[v + "_cd"]), v
        assert r.abort_reason == str(h[v + "_reason"]), v
        assert np.array_equal(r.final_state, h[v + "_final"]), v


def test_oracle_config1_history_bitwise(golden):
    """Config 1 (38,400 points, manish_ad, M 0.63, AoA 2): the full trajectory
    including the abort during iteration 423 at point 27005."""
    h = np.load(os.path.join(golden, "config1_history.npz"))
    c = kf.generate_naca_ogrid("0012", 320, 120, 20.0)
    nb = c.nbr
    o = Oracle(c.x, c.y, c.kind, c.normal_x, c.normal_y, nb.offsets, nb.ids)
    r = o.run(variant="manish_ad", n_iterations=1000, mach=0.63, aoa_deg=2.0, cfl=0.2)
    assert len(r.residual) == 422
    assert np.array_equal(r.residual, h["residual"])
    assert np.array_equal(r.cl, h["cl"]) and np.array_equal(r.cd, h["cd"])
    assert np.array_equal(r.first_order, h["first_order"])
    assert r.diverged and r.abort_reason == str(h["abort_reason"]) == "nonpositive density at point 27005"
    assert np.array_equal(r.final_state[::97], h["final_state_rows"])


def test_oracle_physics_vs_golden(golden):
    g = np.load(os.path.join(golden, "physics.npz"))
    U, dU = g["U"], g["dU"]
    for axis in (0, 1):
        for sign in (0, 1):
            G = np.array([Oracle.split_flux(u, axis, sign) for u in U])
            assert np.array_equal(G, g[f"split_{axis}{sign}"])
            J = np.array([Oracle.jvp_split(u, d, axis, sign, True) for u, d in zip(U, dU)])
            assert np.array_equal(J, g[f"jvp_{axis}{sign}"])
            Ji = np.array([Oracle.jvp_split(u, d, axis, sign, False) for u, d in zip(U, dU)])
            assert np.array_equal(Ji, g[f"ijvp_{axis}{sign}"])
        F = np.array([Oracle.jvp_full(u, d, axis, True) for u, d in zip(U, dU)])
        assert np.array_equal(F, g[f"jvpfull_{axis}"])


def cons(rho, u1, u2, p):
    return np.array([rho, rho * u1, rho * u2, p / (GAMMA - 1.0) + 0.5 * rho * (u1 * u1 + u2 * u2)])


def test_split_flux_known_answers():
    # test_kinetics.cpp:96-104: stationary unit state, mass flux = 1/sqrt(2 pi)
    U = cons(1.0, 0.0, 0.0, 1.0)
    assert Oracle.split_flux(U, 0, 0)[0] == pytest.approx(0.3989422804014327, rel=1e-12)
    assert Oracle.split_flux(U, 0, 1)[0] == pytest.approx(-0.3989422804014327, rel=1e-12)
    # test_kinetics.cpp:106-121: G+ + G- = G
    rng = np.random.default_rng(1234)
    worst = 0.0
    for _ in range(300):
        rho, u1, u2, p = rng.uniform(0.1, 5), rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(0.05, 5)
        U = cons(rho, u1, u2, p)
        for ax in (0, 1):
            s = Oracle.split_flux(U, ax, 0) + Oracle.split_flux(U, ax, 1)
            full = Oracle.jvp_full(U, U, ax, True)  # homogeneous of degree 1: A U = G(U)
            worst = max(worst, np.max(np.abs(s - full)) / max(1.0, np.max(np.abs(full))))
    assert worst <= 1e-13


def test_jvp_known_answers():
    # test_tangent.cpp:73-96 (FD), :98-111 (split sum), :172-190 (errors)
    rng = np.random.default_rng(2024)
    worst_fd = worst_sum = 0.0
    for _ in range(100):
        U = cons(rng.uniform(0.1, 5), rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(0.05, 5))
        d = rng.uniform(-1, 1, 4)
        for ax in (0, 1):
            for sg in (0, 1):
                ex = Oracle.jvp_split(U, d, ax, sg, True)
                h = 1e-6 * np.linalg.norm(U) / np.linalg.norm(d)
                fd = (Oracle.split_flux(U + h * d, ax, sg) - Oracle.split_flux(U - h * d, ax, sg)) / (2 * h)
                worst_fd = max(worst_fd, np.max(np.abs(ex - fd)) / max(1.0, np.max(np.abs(ex))))
            s = Oracle.jvp_split(U, d, ax, 0) + Oracle.jvp_split(U, d, ax, 1)
            full = Oracle.jvp_full(U, d, ax)
            worst_sum = max(worst_sum, np.max(np.abs(s - full)) / max(1.0, np.max(np.abs(full))))
    assert worst_fd <= 1e-8 and worst_sum <= 1e-12
    good = cons(1.0, 0.1, 0.0, 1.0)
    with pytest.raises(Exception, match="increment"):
        Oracle.jvp_split(good, -1.5 * good, 0, 0, exact=False)


def test_oracle_hand_cloud_cross_stencil():
    """test_spatial.cpp:293-345: the cross stencil reduces to +-1/h arms."""
    h = 0.05
    x, y, kind, nx, ny, off, idx = hand_cloud([(0, 0), (h, 0), (-h, 0), (0, h), (0, -h)],
                                              [[1, 2, 3, 4], [0], [0], [0], [0]])
    o = Oracle(x, y, kind, nx, ny, off, idx)
    w, one, _ = o.ls_split(2)  # xneg of point 0 = [2 (dx=-h), 3, 4 (ties)]
    off2, ids2 = o.csr(2)
    assert list(ids2[off2[0]:off2[1]]) == [2, 3, 4]
    assert w[off2[0]] == pytest.approx(-1.0 / h)


@pytest.mark.skipif(not ref_available(), reason="reference build (oracle/_ref) not present")
@pytest.mark.parametrize("spec", [("2412", 65, 9, 11.0), ("0012", 64, 16, 15.0)])
def test_oracle_vs_live_reference(spec):
    ref = Reference.generate(*spec)
    o = oracle_from_reference(ref)
    for w in range(5):
        a, b = ref.csr(w), o.csr(w)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(ref.colors(), o.colors())
    for v in ["anandh", "manish", "manish_ad", "anandh_ad", "explicit"]:
        cfl = 0.05 if v == "explicit" else 0.2
        ra = ref.run(variant=v, n_iterations=25, mach=0.85, aoa_deg=1.0, cfl=cfl)
        rb = o.run(variant=v, n_iterations=25, mach=0.85, aoa_deg=1.0, cfl=cfl)
        assert np.array_equal(ra.residual, rb.residual), v
        assert np.array_equal(ra.final_state, rb.final_state), v
        assert ra.abort_reason == rb.abort_reason, v


@pytest.mark.skipif(not ref_available(), reason="reference build (oracle/_ref) not present")
def test_oracle_vs_live_reference_lattice_and_freestream():
    pts, nbrs = lattice(9, 7)
    x, y, kind, nx, ny, off, idx = hand_cloud(pts, nbrs)
    ref = Reference.from_arrays(x, y, kind, nx, ny, off, idx)
    o = Oracle(x, y, kind, nx, ny, off, idx)
    rng = np.random.default_rng(5)
    U = np.stack([cons(rng.uniform(0.8, 1.2), rng.uniform(0.2, 0.5), rng.uniform(-0.1, 0.1),
                       rng.uniform(0.6, 0.9)) for _ in range(len(x))])
    q = ref.q(U)
    assert np.array_equal(q, o.q(U))
    gx, gy = ref.grads(q, 3)
    hx, hy = o.grads(q, 3)
    assert np.array_equal(gx, hx) and np.array_equal(gy, hy)
    Ra, da = ref.residual(q, gx, gy)
    Rb, db = o.residual(q, gx, gy)
    assert np.array_equal(Ra, Rb) and np.array_equal(da, db)
    Ra, _ = ref.residual(q, gx, gy, first_order=True)
    Rb, _ = o.residual(q, gx, gy, first_order=True)
    assert np.array_equal(Ra, Rb)


def _matrix():
    m = np.load(os.path.join(os.path.dirname(__file__), "golden", "config_matrix.npz"))
    return m, json.loads(str(m["meta"]))


@pytest.mark.parametrize("name", sorted(_matrix()[1]))
def test_oracle_config_matrix_bitwise(name):
    """The restatement over the configuration matrix (n_inner 1/2/4, CFL ramp,
    free-stream BCs, cambered section, convergence/divergence stops, pressure,
    explicit and first-iteration aborts): bitwise the reference fixtures."""
    m, meta = _matrix()
    case = meta[name]
    c = kf.generate_naca_ogrid(*case["cloud"])
    nb = c.nbr
    o = Oracle(c.x, c.y, c.kind, c.normal_x, c.normal_y, nb.offsets, nb.ids)
    r = o.run(**case["cfg"])
    assert len(r.residual) == case["iters"] and r.abort_reason == case["reason"]
    assert np.array_equal(r.residual, m[name + "_residual"])
    assert np.array_equal(r.cl, m[name + "_cl"]) and np.array_equal(r.cd, m[name + "_cd"])
    assert np.array_equal(r.first_order, m[name + "_first_order"])
    assert np.array_equal(r.final_state, m[name + "_final"])


@pytest.mark.parametrize("variant", ["explicit", "anandh", "anandh_ad", "manish", "manish_ad"])
def test_oracle_irregular_cloud_bitwise(golden, variant):
    """Jittered O-grid with random extra neighbours (degrees 5..19, 10
    colours; tests/golden/make_irregular.py), incl. the incremental
    sweep's invalid-increment abort: the restatement is bitwise the
    reference."""
    g = np.load(os.path.join(golden, "irregular_histories.npz"))
    o = Oracle(g["x"], g["y"], g["kind"], g["nx"], g["ny"], g["off"], g["ids"])
    r = o.run(variant=variant, n_iterations=40, mach=0.63, aoa_deg=2.0, cfl=0.05 if variant == "explicit" else 0.2)
    assert r.abort_reason == str(g[variant + "_reason"])
    assert np.array_equal(r.residual, g[variant + "_residual"])
    assert np.array_equal(r.cl, g[variant + "_cl"]) and np.array_equal(r.cd, g[variant + "_cd"])
    assert np.array_equal(r.final_state, g[variant + "_final"])
