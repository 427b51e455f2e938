"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the two CPU checkers.

* ``Reference``: the UNMODIFIED reference solver (``oracle/_ref/libkfref.so``,
  compiled from /root/reference/proj/src by oracle/Makefile, shim in
  oracle/ref_shim.cpp).
* ``Oracle``: the plain-C restatement (``oracle/_build/libkforacle.so``,
  oracle/kf_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module. The product path (paper_2406_07441_b200) never
does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libkfref.so")
ORACLE_SO = os.path.join(HERE, "_build", "libkforacle.so")

VARIANTS = ["explicit", "anandh", "anandh_ad", "manish", "manish_ad"]

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    pass


class _Config(C.Structure):
    _fields_ = [
        ("variant", C.c_int),
        ("cfl", C.c_double),
        ("n_iterations", C.c_int),
        ("n_inner", C.c_int),
        ("mach", C.c_double),
        ("aoa_deg", C.c_double),
        ("convergence_decades", C.c_double),
        ("bc_mode", C.c_int),
        ("cfl_ramp_iters", C.c_int),
        ("cfl_start", C.c_double),
        ("divergence_factor", C.c_double),
    ]


def make_config(variant="manish_ad", cfl=0.2, n_iterations=100, n_inner=3, mach=0.63,
                aoa_deg=0.0, convergence_decades=0.0, bc_mode="physical",
                cfl_ramp_iters=0, cfl_start=0.0, divergence_factor=1e6):
    """Mirror of SolverConfig defaults (driver.hpp:37-52)."""
    return _Config(VARIANTS.index(variant), cfl, n_iterations, n_inner, mach, aoa_deg,
                   convergence_decades, 0 if bc_mode == "physical" else 1,
                   cfl_ramp_iters, cfl_start, divergence_factor)


@dataclass
class RunResult:
    residual: np.ndarray
    cl: np.ndarray
    cd: np.ndarray
    seconds: np.ndarray
    first_order: np.ndarray
    counters: np.ndarray
    sweep: np.ndarray
    final_state: np.ndarray
    diverged: bool
    abort_reason: str
    loop_seconds: float


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class _Lib:
    _cache: dict = {}

    @classmethod
    def get(cls, path):
        if path not in cls._cache:
            if not os.path.exists(path):
                raise OracleError(f"checker library missing: {path} (run make -C oracle)")
            cls._cache[path] = C.CDLL(path)
        return cls._cache[path]


def _err():
    return C.create_string_buffer(512)


class Reference:
    """One reference cloud context (PointCloud + LsCoefficients + SweepPlan)."""

    def __init__(self, handle, lib):
        self._h = handle
        self._lib = lib
        self.n = lib.kfref_n(handle)

    # -- construction -------------------------------------------------------
    @staticmethod
    def lib():
        lib = _Lib.get(REF_SO)
        if not getattr(lib, "_typed", False):
            lib.kfref_generate.restype = C.c_void_p
            lib.kfref_generate.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_double, C.c_char_p, C.c_int]
            lib.kfref_load.restype = C.c_void_p
            lib.kfref_load.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
            lib.kfref_from_arrays.restype = C.c_void_p
            lib.kfref_from_arrays.argtypes = [C.c_int, _dp, _dp, _ip, _dp, _dp, _ip, _ip, C.c_char_p, C.c_int]
            lib.kfref_free.argtypes = [C.c_void_p]
            for f in ("kfref_n", "kfref_n_colors"):
                getattr(lib, f).argtypes = [C.c_void_p]
            lib.kfref_list_nnz.restype = C.c_long
            lib.kfref_list_nnz.argtypes = [C.c_void_p, C.c_int]
            lib.kfref_list.argtypes = [C.c_void_p, C.c_int, _ip, _ip]
            lib.kfref_geometry.argtypes = [C.c_void_p, _dp, _dp, _ip, _dp, _dp]
            lib.kfref_ls_full.argtypes = [C.c_void_p, _dp, _dp, _ip]
            lib.kfref_ls_split.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _ip]
            lib.kfref_flagged.argtypes = [C.c_void_p, C.c_void_p]
            lib.kfref_colors.argtypes = [C.c_void_p, _ip]
            lib.kfref_save.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int]
            lib.kfref_report.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
            lib.kfref_freestream.argtypes = [C.c_double, C.c_double, _dp]
            lib.kfref_q.argtypes = [C.c_void_p, _dp, _dp, C.c_char_p, C.c_int]
            lib.kfref_grads.argtypes = [C.c_void_p, _dp, C.c_int, _dp, _dp]
            lib.kfref_residual.argtypes = [C.c_void_p, _dp, _dp, _dp, C.c_int, _dp, _ip, C.c_char_p, C.c_int]
            lib.kfref_timestep.argtypes = [C.c_void_p, _dp, C.c_double, _dp, C.c_char_p, C.c_int]
            lib.kfref_s_term.argtypes = [C.c_void_p, _dp, _dp, C.c_int, _dp, C.POINTER(C.c_int), C.c_char_p, C.c_int]
            lib.kfref_diagonal.argtypes = [C.c_void_p, _dp, _dp, C.c_int, _dp, C.c_char_p, C.c_int]
            lib.kfref_sweeps.argtypes = [C.c_void_p, _dp, _dp, C.c_void_p, _dp, C.c_int, _dp, _dp, _up, C.c_char_p, C.c_int]
            lib.kfref_bc.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double, C.c_int, C.c_char_p, C.c_int]
            lib.kfref_forces.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p, C.c_char_p, C.c_int]
            lib.kfref_run.argtypes = [C.c_void_p, C.POINTER(_Config), C.POINTER(C.c_int), _dp, _dp, _dp, _dp, _ip, _up, _up, _dp, C.POINTER(C.c_int), C.POINTER(C.c_double), C.c_char_p, C.c_int]
            lib.kfref_num_threads.argtypes = [C.c_int]
            lib.kfref_counters.argtypes = [_up]
            lib.kfref_set_colors.argtypes = [C.c_void_p, _ip]
            lib.kfref_split_flux.argtypes = [_dp, C.c_int, C.c_int, _dp]
            lib.kfref_jvp_split.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int, _dp]
            lib.kfref_jvp_full.argtypes = [_dp, _dp, C.c_int, C.c_int, _dp]
            lib._typed = True
        return lib

    @classmethod
    def generate(cls, digits="0012", n_wall=320, n_radial=120, radius=20.0):
        lib = cls.lib()
        e = _err()
        h = lib.kfref_generate(digits.encode(), n_wall, n_radial, radius, e, 512)
        if not h:
            raise OracleError(e.value.decode())
        return cls(h, lib)

    @classmethod
    def load(cls, path):
        lib = cls.lib()
        e = _err()
        h = lib.kfref_load(str(path).encode(), e, 512)
        if not h:
            raise OracleError(e.value.decode())
        return cls(h, lib)

    @classmethod
    def from_arrays(cls, x, y, kind, nx, ny, off, idx):
        lib = cls.lib()
        e = _err()
        n = len(x)
        h = lib.kfref_from_arrays(n, np.ascontiguousarray(x, np.float64), np.ascontiguousarray(y, np.float64),
                                  np.ascontiguousarray(kind, np.int32), np.ascontiguousarray(nx, np.float64),
                                  np.ascontiguousarray(ny, np.float64), np.ascontiguousarray(off, np.int32),
                                  np.ascontiguousarray(idx, np.int32), e, 512)
        if not h:
            raise OracleError(e.value.decode())
        return cls(h, lib)

    def __del__(self):
        try:
            if self._h:
                self._lib.kfref_free(self._h)
                self._h = None
        except Exception:
            pass

    # -- geometry / ingestion ----------------------------------------------
    def geometry(self):
        n = self.n
        x, y, nx, ny = (np.zeros(n) for _ in range(4))
        kind = np.zeros(n, np.int32)
        self._lib.kfref_geometry(self._h, x, y, kind, nx, ny)
        return x, y, kind, nx, ny

    def csr(self, which):
        """which: 0 nbr, 1 xpos, 2 xneg, 3 ypos, 4 yneg."""
        nnz = self._lib.kfref_list_nnz(self._h, which)
        off = np.zeros(self.n + 1, np.int32)
        idx = np.zeros(max(nnz, 1), np.int32)
        self._lib.kfref_list(self._h, which, off, idx)
        return off, idx[:nnz]

    def ls_full(self):
        nnz = self._lib.kfref_list_nnz(self._h, 0)
        wx = np.zeros(max(nnz, 1)); wy = np.zeros(max(nnz, 1)); kinds = np.zeros(self.n, np.int32)
        self._lib.kfref_ls_full(self._h, wx, wy, kinds)
        return wx[:nnz], wy[:nnz], kinds

    def ls_split(self, which):
        nnz = self._lib.kfref_list_nnz(self._h, which)
        w = np.zeros(max(nnz, 1)); one = np.zeros(self.n); kinds = np.zeros(self.n, np.int32)
        self._lib.kfref_ls_split(self._h, which, w, one, kinds)
        return w[:nnz], one, kinds

    def flagged(self):
        m = self._lib.kfref_flagged(self._h, None)
        out = np.zeros(max(m, 1), np.int32)
        self._lib.kfref_flagged(self._h, out.ctypes.data_as(C.c_void_p))
        return out[:m]

    def report(self):
        ne, ns = C.c_int(), C.c_int()
        self._lib.kfref_report(self._h, None, None, C.byref(ne), C.byref(ns))
        e = np.zeros(max(ne.value, 1), np.int32); s = np.zeros(max(ns.value, 1), np.int32)
        self._lib.kfref_report(self._h, e.ctypes.data_as(C.c_void_p), s.ctypes.data_as(C.c_void_p), C.byref(ne), C.byref(ns))
        return e[:ne.value], s[:ns.value]

    def colors(self):
        c = np.zeros(self.n, np.int32)
        self._lib.kfref_colors(self._h, c)
        return c

    def set_colors(self, color):
        """Run with a caller-supplied colouring (the SweepPlan run_fixed_point
        takes, built by the reference's build_sweep_plan)."""
        bad = self._lib.kfref_set_colors(self._h, np.ascontiguousarray(color, np.int32))
        if bad:
            raise OracleError(f"invalid colouring: {bad} neighbour pairs share a colour")

    def save(self, path):
        e = _err()
        if self._lib.kfref_save(self._h, str(path).encode(), e, 512):
            raise OracleError(e.value.decode())

    # -- stages --------------------------------------------------------------
    @staticmethod
    def freestream(mach, aoa):
        u = np.zeros(4)
        Reference.lib().kfref_freestream(mach, aoa, u)
        return u

    def initial_state(self, mach, aoa, bc_mode="physical"):
        U = np.tile(self.freestream(mach, aoa), (self.n, 1))
        return self.bc(U, mach, aoa, bc_mode)

    def _chk(self, rc, e):
        if rc:
            raise OracleError(e.value.decode())

    def q(self, U):
        e = _err(); q = np.zeros((self.n, 4))
        self._chk(self._lib.kfref_q(self._h, np.ascontiguousarray(U), q, e, 512), e)
        return q

    def grads(self, q, n_inner=3):
        qx = np.zeros((self.n, 4)); qy = np.zeros((self.n, 4))
        self._lib.kfref_grads(self._h, np.ascontiguousarray(q), n_inner, qx, qy)
        return qx, qy

    def residual(self, q, qx, qy, first_order=False):
        e = _err(); R = np.zeros((self.n, 4)); dem = np.zeros(self.n, np.int32)
        self._chk(self._lib.kfref_residual(self._h, np.ascontiguousarray(q), np.ascontiguousarray(qx),
                                           np.ascontiguousarray(qy), int(first_order), R, dem, e, 512), e)
        return R, dem

    def timestep(self, U, cfl):
        e = _err(); dt = np.zeros(self.n)
        self._chk(self._lib.kfref_timestep(self._h, np.ascontiguousarray(U), cfl, dt, e, 512), e)
        return dt

    def s_term(self, U, dU_prev, exact=True):
        e = _err(); S = np.zeros((self.n, 4)); nf = C.c_int()
        self._chk(self._lib.kfref_s_term(self._h, np.ascontiguousarray(U), np.ascontiguousarray(dU_prev),
                                         int(exact), S, C.byref(nf), e, 512), e)
        return S, nf.value

    def diagonal(self, U, dt, variant):
        e = _err(); d = np.zeros(self.n)
        self._chk(self._lib.kfref_diagonal(self._h, np.ascontiguousarray(U), np.ascontiguousarray(dt),
                                           VARIANTS.index(variant), d, e, 512), e)
        return d

    def sweeps(self, U, R, S, d, exact=True):
        e = _err(); ds = np.zeros((self.n, 4)); du = np.zeros((self.n, 4)); cnt = np.zeros(5, np.uint64)
        Sp = None if S is None else np.ascontiguousarray(S)
        self._chk(self._lib.kfref_sweeps(self._h, np.ascontiguousarray(U), np.ascontiguousarray(R),
                                         None if Sp is None else Sp.ctypes.data_as(C.c_void_p),
                                         np.ascontiguousarray(d), int(exact), ds, du, cnt, e, 512), e)
        return ds, du, cnt

    def bc(self, U, mach, aoa, bc_mode="physical"):
        e = _err(); V = np.array(U, dtype=np.float64, order="C", copy=True)
        self._chk(self._lib.kfref_bc(self._h, V, mach, aoa, 0 if bc_mode == "physical" else 1, e, 512), e)
        return V

    def forces(self, U, mach, aoa, n_wall=None):
        e = _err(); cl = C.c_double(); cd = C.c_double()
        self._chk(self._lib.kfref_forces(self._h, np.ascontiguousarray(U), mach, aoa, C.byref(cl), C.byref(cd),
                                         None, e, 512), e)
        return cl.value, cd.value

    def run(self, **cfg) -> RunResult:
        c = make_config(**cfg)
        m = c.n_iterations
        res, cl, cd, sec = (np.zeros(m) for _ in range(4))
        fo = np.zeros(m, np.int32)
        cnt = np.zeros(m * 5, np.uint64); sw = np.zeros(m * 5, np.uint64)
        fs = np.zeros((self.n, 4))
        nd = C.c_int(); dv = C.c_int(); ls = C.c_double(); e = _err()
        rc = self._lib.kfref_run(self._h, C.byref(c), C.byref(nd), res, cl, cd, sec, fo, cnt, sw, fs,
                                 C.byref(dv), C.byref(ls), e, 512)
        if rc:
            raise OracleError(e.value.decode())
        k = nd.value
        return RunResult(res[:k], cl[:k], cd[:k], sec[:k], fo[:k], cnt.reshape(m, 5)[:k],
                         sw.reshape(m, 5)[:k], fs, bool(dv.value), e.value.decode(), ls.value)

    @staticmethod
    def num_threads(n=0):
        return Reference.lib().kfref_num_threads(n)


class _Err(C.Structure):
    _fields_ = [("code", C.c_int), ("point", C.c_int), ("msg", C.c_char * 192)]


class Oracle:
    """The plain-C restatement (oracle/kf_oracle.c) over the same arrays."""

    def __init__(self, x, y, kind, nx, ny, off, idx):
        lib = self.lib()
        self._lib = lib
        self.n = len(x)
        self._keep = [np.ascontiguousarray(a, t) for a, t in
                      ((x, np.float64), (y, np.float64), (kind, np.int32), (nx, np.float64),
                       (ny, np.float64), (off, np.int32), (idx, np.int32))]
        self._h = lib.kfo_cloud_new(self.n, *self._keep)

    @staticmethod
    def lib():
        lib = _Lib.get(ORACLE_SO)
        if not getattr(lib, "_typed", False):
            lib.kfo_cloud_new.restype = C.c_void_p
            lib.kfo_cloud_new.argtypes = [C.c_int, _dp, _dp, _ip, _dp, _dp, _ip, _ip]
            lib.kfo_cloud_free.argtypes = [C.c_void_p]
            lib.kfo_n_colors.argtypes = [C.c_void_p]
            lib.kfo_list_nnz.restype = C.c_long
            lib.kfo_list_nnz.argtypes = [C.c_void_p, C.c_int]
            lib.kfo_list.argtypes = [C.c_void_p, C.c_int, _ip, _ip]
            lib.kfo_ls_full.argtypes = [C.c_void_p, _dp, _dp, _ip]
            lib.kfo_ls_split.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _ip]
            lib.kfo_flagged.argtypes = [C.c_void_p, C.c_void_p]
            lib.kfo_colors.argtypes = [C.c_void_p, _ip]
            lib.kfo_report.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int), C.c_void_p, C.POINTER(C.c_int)]
            lib.kfo_freestream.argtypes = [C.c_double, C.c_double, _dp]
            E = C.POINTER(_Err)
            lib.kfo_q.argtypes = [C.c_void_p, _dp, _dp, E]
            lib.kfo_grads.argtypes = [C.c_void_p, _dp, C.c_int, _dp, _dp]
            lib.kfo_residual.argtypes = [C.c_void_p, _dp, _dp, _dp, C.c_int, _dp, _ip, E]
            lib.kfo_timestep.argtypes = [C.c_void_p, _dp, C.c_double, _dp, E]
            lib.kfo_s_term.argtypes = [C.c_void_p, _dp, _dp, C.c_int, _dp, C.POINTER(C.c_int), E]
            lib.kfo_diagonal.argtypes = [C.c_void_p, _dp, _dp, C.c_int, _dp, E]
            lib.kfo_sweeps.argtypes = [C.c_void_p, _dp, _dp, C.c_void_p, _dp, C.c_int, _dp, _dp, E]
            lib.kfo_bc.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double, C.c_int, E]
            lib.kfo_forces.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double), E]
            lib.kfo_run.argtypes = [C.c_void_p, C.POINTER(_Config), C.POINTER(C.c_int), _dp, _dp, _dp, _ip, _dp, C.POINTER(C.c_int), C.c_char_p, C.c_int]
            lib.kfo_split_flux.argtypes = [_dp, C.c_int, C.c_int, _dp]
            lib.kfo_jvp_split.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int, _dp]
            lib.kfo_jvp_full.argtypes = [_dp, _dp, C.c_int, C.c_int, _dp]
            lib._typed = True
        return lib

    def __del__(self):
        try:
            if self._h:
                self._lib.kfo_cloud_free(self._h)
                self._h = None
        except Exception:
            pass

    def _chk(self, rc, e):
        if rc:
            raise OracleError(e.msg.decode())

    def csr(self, which):
        nnz = self._lib.kfo_list_nnz(self._h, which)
        off = np.zeros(self.n + 1, np.int32); idx = np.zeros(max(nnz, 1), np.int32)
        self._lib.kfo_list(self._h, which, off, idx)
        return off, idx[:nnz]

    def ls_full(self):
        nnz = self._lib.kfo_list_nnz(self._h, 0)
        wx = np.zeros(max(nnz, 1)); wy = np.zeros(max(nnz, 1)); k = np.zeros(self.n, np.int32)
        self._lib.kfo_ls_full(self._h, wx, wy, k)
        return wx[:nnz], wy[:nnz], k

    def ls_split(self, which):
        nnz = self._lib.kfo_list_nnz(self._h, which)
        w = np.zeros(max(nnz, 1)); one = np.zeros(self.n); k = np.zeros(self.n, np.int32)
        self._lib.kfo_ls_split(self._h, which, w, one, k)
        return w[:nnz], one, k

    def flagged(self):
        m = self._lib.kfo_flagged(self._h, None)
        out = np.zeros(max(m, 1), np.int32)
        self._lib.kfo_flagged(self._h, out.ctypes.data_as(C.c_void_p))
        return out[:m]

    def report(self):
        ne, ns = C.c_int(), C.c_int()
        e = np.zeros(self.n + 1, np.int32); s = np.zeros(self.n + 1, np.int32)
        self._lib.kfo_report(self._h, e.ctypes.data_as(C.c_void_p), C.byref(ne), s.ctypes.data_as(C.c_void_p), C.byref(ns))
        return e[:ne.value], s[:ns.value]

    def colors(self):
        c = np.zeros(self.n, np.int32)
        self._lib.kfo_colors(self._h, c)
        return c

    @staticmethod
    def freestream(mach, aoa):
        u = np.zeros(4)
        Oracle.lib().kfo_freestream(mach, aoa, u)
        return u

    def initial_state(self, mach, aoa, bc_mode="physical"):
        U = np.tile(self.freestream(mach, aoa), (self.n, 1))
        return self.bc(U, mach, aoa, bc_mode)

    def q(self, U):
        e = _Err(); q = np.zeros((self.n, 4))
        self._chk(self._lib.kfo_q(self._h, np.ascontiguousarray(U), q, C.byref(e)), e)
        return q

    def grads(self, q, n_inner=3):
        qx = np.zeros((self.n, 4)); qy = np.zeros((self.n, 4))
        self._lib.kfo_grads(self._h, np.ascontiguousarray(q), n_inner, qx, qy)
        return qx, qy

    def residual(self, q, qx, qy, first_order=False):
        e = _Err(); R = np.zeros((self.n, 4)); dem = np.zeros(self.n, np.int32)
        self._chk(self._lib.kfo_residual(self._h, np.ascontiguousarray(q), np.ascontiguousarray(qx),
                                         np.ascontiguousarray(qy), int(first_order), R, dem, C.byref(e)), e)
        return R, dem

    def timestep(self, U, cfl):
        e = _Err(); dt = np.zeros(self.n)
        self._chk(self._lib.kfo_timestep(self._h, np.ascontiguousarray(U), cfl, dt, C.byref(e)), e)
        return dt

    def s_term(self, U, dU_prev, exact=True):
        e = _Err(); S = np.zeros((self.n, 4)); nf = C.c_int()
        self._chk(self._lib.kfo_s_term(self._h, np.ascontiguousarray(U), np.ascontiguousarray(dU_prev),
                                       int(exact), S, C.byref(nf), C.byref(e)), e)
        return S, nf.value

    def diagonal(self, U, dt, variant):
        e = _Err(); d = np.zeros(self.n)
        self._chk(self._lib.kfo_diagonal(self._h, np.ascontiguousarray(U), np.ascontiguousarray(dt),
                                         VARIANTS.index(variant), d, C.byref(e)), e)
        return d

    def sweeps(self, U, R, S, d, exact=True):
        e = _Err(); ds = np.zeros((self.n, 4)); du = np.zeros((self.n, 4))
        Sp = None if S is None else np.ascontiguousarray(S)
        self._chk(self._lib.kfo_sweeps(self._h, np.ascontiguousarray(U), np.ascontiguousarray(R),
                                       None if Sp is None else Sp.ctypes.data_as(C.c_void_p),
                                       np.ascontiguousarray(d), int(exact), ds, du, C.byref(e)), e)
        return ds, du

    def bc(self, U, mach, aoa, bc_mode="physical"):
        e = _Err(); V = np.array(U, dtype=np.float64, order="C", copy=True)
        self._chk(self._lib.kfo_bc(self._h, V, mach, aoa, 0 if bc_mode == "physical" else 1, C.byref(e)), e)
        return V

    def forces(self, U, mach, aoa):
        e = _Err(); cl = C.c_double(); cd = C.c_double()
        self._chk(self._lib.kfo_forces(self._h, np.ascontiguousarray(U), mach, aoa, C.byref(cl), C.byref(cd), C.byref(e)), e)
        return cl.value, cd.value

    def run(self, **cfg) -> RunResult:
        c = make_config(**cfg)
        m = c.n_iterations
        res, cl, cd = (np.zeros(m) for _ in range(3))
        fo = np.zeros(m, np.int32)
        fs = np.zeros((self.n, 4))
        nd = C.c_int(); dv = C.c_int(); e = C.create_string_buffer(512)
        rc = self._lib.kfo_run(self._h, C.byref(c), C.byref(nd), res, cl, cd, fo, fs, C.byref(dv), e, 512)
        if rc:
            raise OracleError(e.value.decode())
        k = nd.value
        return RunResult(res[:k], cl[:k], cd[:k], np.zeros(k), fo[:k], np.zeros((k, 5), np.uint64),
                         np.zeros((k, 5), np.uint64), fs, bool(dv.value), e.value.decode(), 0.0)

    # point physics
    @staticmethod
    def split_flux(U, axis, sign):
        G = np.zeros(4)
        if Oracle.lib().kfo_split_flux(np.ascontiguousarray(U, np.float64), axis, sign, G):
            raise OracleError("invalid state")
        return G

    @staticmethod
    def jvp_split(U, dU, axis, sign, exact=True):
        o = np.zeros(4)
        rc = Oracle.lib().kfo_jvp_split(np.ascontiguousarray(U, np.float64), np.ascontiguousarray(dU, np.float64), axis, sign, int(exact), o)
        if rc:
            raise OracleError("invalid state" if rc == 1 else "invalid increment")
        return o

    @staticmethod
    def jvp_full(U, dU, axis, exact=True):
        o = np.zeros(4)
        rc = Oracle.lib().kfo_jvp_full(np.ascontiguousarray(U, np.float64), np.ascontiguousarray(dU, np.float64), axis, int(exact), o)
        if rc:
            raise OracleError("invalid state" if rc == 1 else "invalid increment")
        return o


def oracle_from_reference(ref: Reference) -> Oracle:
    """Oracle built on exactly the reference cloud's raw arrays."""
    x, y, kind, nx, ny = ref.geometry()
    off, idx = ref.csr(0)
    return Oracle(x, y, kind, nx, ny, off, idx)
