"""The C-ABI library (CPU only): it loads, exports every symbol include/kf.h
declares, and the device entry points fail loudly (no CPU fallback) when no
GPU is present.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2406_07441_b200 as kf
from paper_2406_07441_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "kf.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kf_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_what_binding_expects():
    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_version_and_defaults():
    assert "sm_100a" in kf.version()
    cfg = _lib.Config()
    _lib.lib.kf_config_default(C.byref(cfg))
    # SolverConfig defaults, driver.hpp:37-52
    assert (cfg.variant, cfg.cfl, cfg.n_iterations, cfg.n_inner, cfg.mach_inf) == (0, 0.2, 100, 3, 0.63)
    assert cfg.divergence_factor == 1e6 and cfg.bc_mode == 0


def test_preconditions_raise_like_reference():
    c = kf.generate_naca_ogrid("0012", 32, 8, 10.0)
    with pytest.raises(kf.ConfigError, match="cfl must be positive"):
        kf.Solver(c, kf.SolverConfig(cfl=0.0))
    with pytest.raises(kf.ConfigError, match="n_iterations"):
        kf.Solver(c, kf.SolverConfig(n_iterations=0))


def test_no_gpu_fails_loudly(has_gpu):
    if has_gpu:
        pytest.skip("GPU present")
    c = kf.generate_naca_ogrid("0012", 32, 8, 10.0)
    with pytest.raises(kf.CudaError, match="no CUDA device"):
        kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD))
    with pytest.raises(kf.CudaError):
        kf.split_flux(np.array([[1.0, 0.1, 0.0, 2.5]]), 0, 0)


def test_singular_interior_stencil_refused():
    # driver.cpp:198-201: an interior point with a singular LS stencil aborts setup
    from util import hand_cloud
    c = kf.PointCloud.from_arrays(*hand_cloud([(0, 0), (1, 1), (2, 2), (-1, -1)],
                                              [[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]]))
    with pytest.raises(kf.KinfreeError, match="singular least-squares stencil"):
        kf.Solver(c, kf.SolverConfig(variant=kf.SolverVariant.ManishAD))


def test_create_rank_validates_arguments():
    import ctypes as C
    from paper_2406_07441_b200 import _lib
    c = kf.generate_naca_ogrid("0012", 32, 8, 10.0)
    cfg = kf.SolverConfig(variant=kf.SolverVariant.ManishAD).to_c()
    h = C.c_void_p()
    st = _lib.lib.kf_create_rank(c.handle, C.byref(cfg), 2, 0, 0, None, C.byref(h))
    assert st.code == _lib.KF_CONFIG and b"NCCL unique id" in st.reason
    st = _lib.lib.kf_create_rank(c.handle, C.byref(cfg), 2, 2, 0, b"x" * 128, C.byref(h))
    assert st.code == _lib.KF_CONFIG and b"rank out of range" in st.reason


def test_create_rank_host_validates_arguments():
    """kf_create_rank_host: missing callbacks and bad ranks are configuration
    errors (checked before any device work, so this runs without a GPU)."""
    import ctypes as C
    from paper_2406_07441_b200 import _lib
    c = kf.generate_naca_ogrid("0012", 32, 8, 10.0)
    cfg = kf.SolverConfig(variant=kf.SolverVariant.ManishAD).to_c()
    h = C.c_void_p()
    ex = _lib.EXCHANGE_FN(lambda *a: 0)
    ar = _lib.ALLREDUCE_FN(lambda *a: 0)
    st = _lib.lib.kf_create_rank_host(c.handle, C.byref(cfg), 2, 0, 0, _lib.EXCHANGE_FN(), ar, None, C.byref(h))
    assert st.code == _lib.KF_CONFIG and b"callback" in st.reason
    st = _lib.lib.kf_create_rank_host(c.handle, C.byref(cfg), 2, 5, 0, ex, ar, None, C.byref(h))
    assert st.code == _lib.KF_CONFIG and b"rank out of range" in st.reason


def test_step_host_validates_buffers_before_native_code():
    """Solver.step_host / step_host_batch check dtype, shape and contiguity of
    the caller's arrays before any pointer reaches kf_step_host (no device
    needed: the checks fail first)."""
    s = object.__new__(kf.Solver)
    s.n = 6
    U = np.zeros((6, 4))
    for bad in [dict(dU_prev_in=None), dict(U_in=np.zeros((5, 4))),
                dict(U_out=np.zeros((6, 4), np.float32)), dict(U_out=np.zeros((6, 8))[:, ::2]),
                dict(dU_out=np.zeros((6, 4), np.int64))]:
        args = dict(U_in=U, dU_prev_in=U, U_out=None, dU_out=None)
        args.update(bad)
        with pytest.raises(kf.ConfigError):
            s.step_host(**args)
    with pytest.raises(kf.ConfigError):
        s.step_host_batch([U], [U], [np.zeros((6, 4), np.float32)])
    with pytest.raises(kf.ConfigError):
        s.step_host_batch([U, U], [U], [U, U])
