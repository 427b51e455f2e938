"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs /root/reference and `make -C oracle ref`):

    python tests/golden/make_golden.py

The fixtures travel with the repo so the GPU box (which has no
/root/reference) can pin both the C restatement (oracle/) and the CUDA path
against the reference's own outputs:

* ``ingest_hashes.json``  sha256 of every ingested array (geometry, CSR
  stencils, LS weights, colours) for the BASELINE.json config clouds.
* ``stages_<variant>.npz``  per-stage inputs/outputs of one iteration on a
  48x12 O-grid after 8 iterations of that variant (driver.cpp:229-252).
* ``config1_history.npz``  the config-1 run (naca0012 320x120, M 0.63,
  AoA 2, manish_ad, CFL 0.2, 1000 iterations): residual/CL/CD history and
  the abort record.
* ``physics.npz``  split fluxes and JVPs on the reference tests' random
  state distribution (oracles.cpp:193-203).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from refpy import Reference  # noqa: E402

CLOUDS = {
    "config1": ("0012", 320, 120, 20.0),
    "config2": ("0012", 1280, 500, 20.0),
    "small": ("0012", 48, 12, 12.0),
    "odd": ("2412", 65, 9, 11.0),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ingest_hashes(ref: Reference):
    x, y, kind, nx, ny = ref.geometry()
    out = {"n": int(ref.n), "x": sha(x), "y": sha(y), "kind": sha(kind.astype(np.int32)),
           "nx": sha(nx), "ny": sha(ny)}
    for w, name in enumerate(["nbr", "xpos", "xneg", "ypos", "yneg"]):
        off, idx = ref.csr(w)
        out[name + "_off"] = sha(off)
        out[name + "_idx"] = sha(idx)
    wx, wy, k = ref.ls_full()
    out.update(wx=sha(wx), wy=sha(wy), full_kind=sha(k))
    for w, name in [(1, "xpos"), (2, "xneg"), (3, "ypos"), (4, "yneg")]:
        a, b, kk = ref.ls_split(w)
        out[name + "_w"] = sha(a)
        out[name + "_one"] = sha(b)
        out[name + "_kind"] = sha(kk)
    out["flagged"] = sha(ref.flagged())
    out["color"] = sha(ref.colors())
    out["n_colors"] = int(ref.lib().kfref_n_colors(ref._h))
    return out


def stage_vectors(ref: Reference, variant: str, mach=0.63, aoa=2.0, warm=8, cfl=0.2):
    res = ref.run(variant=variant, n_iterations=warm, mach=mach, aoa_deg=aoa, cfl=cfl)
    assert not res.diverged, res.abort_reason
    U = res.final_state
    # dU_prev of the last warm iteration: rerun warm-1 iterations and difference
    # is not available through the public API, so use one extra reference
    # iteration's sweep output as the next dU_prev instead.
    q = ref.q(U)
    qx, qy = ref.grads(q, 3)
    R, dem = ref.residual(q, qx, qy)
    dt = ref.timestep(U, cfl)
    out = dict(U=U, q=q, qx=qx, qy=qy, R=R, demoted=dem, dt=dt, cfl=np.array(cfl),
               mach=np.array(mach), aoa=np.array(aoa))
    if variant != "explicit":
        exact = variant.endswith("_ad")
        with_s = variant.startswith("manish")
        # a nonzero dU_prev: the sweep result of this state with S=0
        d0 = ref.diagonal(U, dt, variant)
        _, dU_prev, _ = ref.sweeps(U, R, None, d0, exact)
        S = ref.s_term(U, dU_prev, exact)[0] if with_s else None
        d = ref.diagonal(U, dt, variant)
        dUs, dU, cnt = ref.sweeps(U, R, S, d, exact)
        Unew = ref.bc(U + dU, mach, aoa)
        cl, cd = ref.forces(Unew, mach, aoa)
        out.update(dU_prev=dU_prev, diag=d, dU_star=dUs, dU=dU, U_next=Unew,
                   cl=np.array(cl), cd=np.array(cd), sweep_counts=cnt)
        if with_s:
            out["S"] = S
    return out


def main():
    hashes = {}
    for name, spec in CLOUDS.items():
        ref = Reference.generate(*spec)
        hashes[name] = ingest_hashes(ref)
        hashes[name]["spec"] = list(spec)
        print("ingest", name, ref.n)
    with open(os.path.join(HERE, "ingest_hashes.json"), "w") as f:
        json.dump(hashes, f, indent=1, sort_keys=True)

    small = Reference.generate(*CLOUDS["small"])
    for v in ["explicit", "anandh", "anandh_ad", "manish", "manish_ad"]:
        cfl = 0.05 if v == "explicit" else 0.2
        np.savez_compressed(os.path.join(HERE, f"stages_{v}.npz"),
                            **stage_vectors(small, v, cfl=cfl))
        print("stages", v)

    ref = Reference.generate(*CLOUDS["config1"])
    res = ref.run(variant="manish_ad", n_iterations=1000, mach=0.63, aoa_deg=2.0, cfl=0.2)
    np.savez_compressed(os.path.join(HERE, "config1_history.npz"), residual=res.residual, cl=res.cl,
                        cd=res.cd, first_order=res.first_order, sweep=res.sweep,
                        counters=res.counters, diverged=np.array(res.diverged),
                        abort_reason=np.array(res.abort_reason),
                        final_state_sha=np.array(sha(res.final_state)),
                        final_state_rows=res.final_state[::97].copy(),
                        state400_rows=ref.run(variant="manish_ad", n_iterations=400, mach=0.63,
                                              aoa_deg=2.0, cfl=0.2).final_state[::97].copy())
    print("config1", len(res.residual), res.abort_reason)

    # short histories of every variant on the small cloud (counters included)
    hist = {}
    for v in ["explicit", "anandh", "anandh_ad", "manish", "manish_ad"]:
        cfl = 0.05 if v == "explicit" else 0.2
        r = small.run(variant=v, n_iterations=60, mach=0.63, aoa_deg=2.0, cfl=cfl)
        hist[v + "_residual"] = r.residual
        hist[v + "_cl"] = r.cl
        hist[v + "_cd"] = r.cd
        hist[v + "_counters"] = r.counters
        hist[v + "_sweep"] = r.sweep
        hist[v + "_reason"] = np.array(r.abort_reason)
        hist[v + "_final"] = r.final_state
    np.savez_compressed(os.path.join(HERE, "small_histories.npz"), **hist)

    # point physics on the reference tests' state distribution
    rng = np.random.default_rng(1234)
    m = 256
    rho = rng.uniform(0.1, 5.0, m)
    u1 = rng.uniform(-3, 3, m)
    u2 = rng.uniform(-3, 3, m)
    p = rng.uniform(0.05, 5.0, m)
    U = np.stack([rho, rho * u1, rho * u2, p / 0.3999999999999999 + 0.5 * rho * (u1 * u1 + u2 * u2)], 1)
    dU = rng.uniform(-1, 1, (m, 4)) * 1e-3 * np.abs(U).max(1, keepdims=True)
    lib = Reference.lib()
    phys = {"U": U, "dU": dU}
    for axis in (0, 1):
        for sign in (0, 1):
            G = np.zeros((m, 4))
            J = np.zeros((m, 4))
            Ji = np.zeros((m, 4))
            for t in range(m):
                g = np.zeros(4)
                lib.kfref_split_flux(U[t], axis, sign, g)
                G[t] = g
                lib.kfref_jvp_split(U[t], dU[t], axis, sign, 1, g)
                J[t] = g
                lib.kfref_jvp_split(U[t], dU[t], axis, sign, 0, g)
                Ji[t] = g
            phys[f"split_{axis}{sign}"] = G
            phys[f"jvp_{axis}{sign}"] = J
            phys[f"ijvp_{axis}{sign}"] = Ji
        F = np.zeros((m, 4))
        for t in range(m):
            g = np.zeros(4)
            lib.kfref_jvp_full(U[t], dU[t], axis, 1, g)
            F[t] = g
        phys[f"jvpfull_{axis}"] = F
    np.savez_compressed(os.path.join(HERE, "physics.npz"), **phys)
    print("physics done")


if __name__ == "__main__":
    main()
