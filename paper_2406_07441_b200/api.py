"""Python mirror of the reference kinfree API over libkf.so.

Names, argument meaning and error behaviour follow the reference C++ headers
so that callers (and the parity tests) read like the reference's own code:

=====================================  =========================================
this module                            reference
=====================================  =========================================
``generate_naca_ogrid``                pointcloud.hpp:59-60
``load_cloud`` / ``save_cloud``        pointcloud.hpp:65-67
``build_ls_coefficients``              spatial.hpp:59
``color_points`` / ``build_sweep_plan`` coloring.hpp:34-36
``SolverVariant`` / ``SolverConfig``   implicit.hpp:35, driver.hpp:37-52
``IterationRecord`` / ``RunHistory``   driver.hpp:54-73
``run_fixed_point``                    driver.hpp:101-106 (the drop-in seam)
``Solver.q/grads/residual/lusgs/...``  per-stage hooks of driver.cpp:229-252
=====================================  =========================================

All compute runs in the CUDA kernels of libkf.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L

lib = L.lib


# ------------------------------------------------------------------ errors
class KinfreeError(RuntimeError):
    def __init__(self, status):
        if isinstance(status, str):  # raised by the Python layer itself
            self.code = {ConfigError: L.KF_CONFIG}.get(type(self), L.KF_RUNTIME)
            self.point, self.iteration, self.reason = -1, 0, status
        else:
            self.code = status.code
            self.point = status.point
            self.iteration = status.iteration
            self.reason = status.reason.decode(errors="replace")
        super().__init__(self.reason)


class InvalidStateError(KinfreeError):
    """invalid_state_error (state.hpp:67-79)."""


class InvalidIncrementError(InvalidStateError):
    """invalid_increment_error (tangent.hpp:28-31)."""


class ConfigError(KinfreeError, ValueError):
    """std::invalid_argument / config_error."""


class CudaError(KinfreeError):
    pass


def _check(st):
    if st.code == L.KF_OK:
        return
    cls = {L.KF_INVALID_STATE: InvalidStateError, L.KF_INVALID_INCREMENT: InvalidIncrementError,
           L.KF_CONFIG: ConfigError, L.KF_CUDA: CudaError}.get(st.code, KinfreeError)
    raise cls(st)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------- point clouds
class PointKind(enum.IntEnum):
    Wall = 0
    Interior = 1
    Outer = 2


@dataclass
class Csr:
    offsets: np.ndarray
    ids: np.ndarray

    def __getitem__(self, p):
        return self.ids[self.offsets[p]:self.offsets[p + 1]]


class PointCloud:
    """Ingested cloud (pointcloud.hpp:28-46) held by libkf."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            lib.kf_cloud_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def n(self) -> int:
        return lib.kf_cloud_n(self._h)

    def _geometry(self):
        n = self.n()
        x, y, nx, ny = (np.zeros(n) for _ in range(4))
        kind = np.zeros(n, np.int32)
        lib.kf_cloud_geometry(self._h, x, y, kind, nx, ny)
        return x, y, kind, nx, ny

    @property
    def x(self):
        return self._geometry()[0]

    @property
    def y(self):
        return self._geometry()[1]

    @property
    def kind(self):
        return self._geometry()[2]

    @property
    def normal_x(self):
        return self._geometry()[3]

    @property
    def normal_y(self):
        return self._geometry()[4]

    def count(self, kind: PointKind) -> int:
        return int(np.count_nonzero(self.kind == int(kind)))

    def _list(self, which) -> Csr:
        nnz = lib.kf_cloud_list_nnz(self._h, which)
        off = np.zeros(self.n() + 1, np.int32)
        idx = np.zeros(max(nnz, 1), np.int32)
        lib.kf_cloud_list(self._h, which, off, idx)
        return Csr(off, idx[:nnz])

    @property
    def nbr(self) -> Csr:
        return self._list(0)

    @property
    def xpos(self) -> Csr:
        return self._list(1)

    @property
    def xneg(self) -> Csr:
        return self._list(2)

    @property
    def ypos(self) -> Csr:
        return self._list(3)

    @property
    def yneg(self) -> Csr:
        return self._list(4)

    @property
    def wall_ids(self):
        return np.flatnonzero(self.kind == 0).astype(np.int32)

    @property
    def interior_ids(self):
        return np.flatnonzero(self.kind == 1).astype(np.int32)

    @property
    def outer_ids(self):
        return np.flatnonzero(self.kind == 2).astype(np.int32)

    @property
    def stencil_report(self):
        ne, ns = C.c_int(), C.c_int()
        lib.kf_cloud_report(self._h, None, C.byref(ne), None, C.byref(ns))
        e = np.zeros(max(ne.value, 1), np.int32)
        s = np.zeros(max(ns.value, 1), np.int32)
        lib.kf_cloud_report(self._h, _ptr(e), C.byref(ne), _ptr(s), C.byref(ns))
        return StencilReport(e[:ne.value], s[:ns.value])

    @classmethod
    def from_arrays(cls, x, y, kind, normal_x, normal_y, nbr_offsets, nbr_ids):
        h = C.c_void_p()
        _check(lib.kf_cloud_from_arrays(len(x), _f64(x), _f64(y), np.ascontiguousarray(kind, np.int32),
                                        _f64(normal_x), _f64(normal_y),
                                        np.ascontiguousarray(nbr_offsets, np.int32),
                                        np.ascontiguousarray(nbr_ids, np.int32), C.byref(h)))
        return cls(h.value)


@dataclass
class StencilReport:
    empty_points: np.ndarray
    singular_points: np.ndarray

    def clean(self):
        return len(self.empty_points) == 0 and len(self.singular_points) == 0


def generate_naca_ogrid(naca_digits: str, n_wall: int, n_radial: int,
                        far_field_radius: float) -> PointCloud:
    h = C.c_void_p()
    _check(lib.kf_cloud_generate_naca(naca_digits.encode(), n_wall, n_radial, far_field_radius,
                                      C.byref(h)))
    return PointCloud(h.value)


def load_cloud(path) -> PointCloud:
    h = C.c_void_p()
    _check(lib.kf_cloud_load(str(path).encode(), C.byref(h)))
    return PointCloud(h.value)


def save_cloud(cloud: PointCloud, path, binary=False) -> None:
    """save_cloud (pointcloud.cpp:383-401); binary=True writes the SoA cache
    that load_cloud recognises (bulk reads instead of the text parser)."""
    _check((lib.kf_cloud_save_binary if binary else lib.kf_cloud_save)(cloud.handle, str(path).encode()))


@dataclass
class LsCoefficients:
    """LsCoefficients (spatial.hpp:44-57) in CSR form."""
    full_wx: np.ndarray
    full_wy: np.ndarray
    full_kind: np.ndarray
    split_w: dict
    ls_one: dict
    split_kind: dict
    flagged: np.ndarray


def build_ls_coefficients(cloud: PointCloud) -> LsCoefficients:
    n = cloud.n()
    nnz = lib.kf_cloud_list_nnz(cloud.handle, 0)
    wx, wy = np.zeros(max(nnz, 1)), np.zeros(max(nnz, 1))
    kinds = np.zeros(n, np.int32)
    lib.kf_cloud_ls_full(cloud.handle, wx, wy, kinds)
    sw, one, sk = {}, {}, {}
    for which, name in ((1, "xpos"), (2, "xneg"), (3, "ypos"), (4, "yneg")):
        m = lib.kf_cloud_list_nnz(cloud.handle, which)
        w, o, k = np.zeros(max(m, 1)), np.zeros(n), np.zeros(n, np.int32)
        lib.kf_cloud_ls_split(cloud.handle, which, w, o, k)
        sw[name], one[name], sk[name] = w[:m], o, k
    m = lib.kf_cloud_flagged(cloud.handle, None)
    fl = np.zeros(max(m, 1), np.int32)
    lib.kf_cloud_flagged(cloud.handle, _ptr(fl))
    return LsCoefficients(wx[:nnz], wy[:nnz], kinds, sw, one, sk, fl[:m])


@dataclass
class ColorAssignment:
    color: np.ndarray  # 1-based
    n_colors: int


@dataclass
class SweepPlan:
    groups: List[np.ndarray]
    color_of: np.ndarray


def color_points(cloud: PointCloud) -> ColorAssignment:
    c = np.zeros(cloud.n(), np.int32)
    lib.kf_cloud_colors(cloud.handle, c)
    return ColorAssignment(c, int(lib.kf_cloud_n_colors(cloud.handle)))


def build_sweep_plan(colors: ColorAssignment) -> SweepPlan:
    groups = [np.flatnonzero(colors.color == g + 1).astype(np.int32) for g in range(colors.n_colors)]
    return SweepPlan(groups, colors.color.copy())


def set_colors(cloud: PointCloud, color_of) -> None:
    """Adopt an external SweepPlan.color_of (must be a valid colouring)."""
    _check(lib.kf_cloud_set_colors(cloud.handle, np.ascontiguousarray(color_of, np.int32)))


def color_points_device(cloud: PointCloud, mode: str = "ldf", seed: int = 1, device: int = 0) -> ColorAssignment:
    """Sweep-ordering variant: a Jones-Plassmann
    colouring computed on the GPU replaces the cloud's greedy colouring
    (color_points, coloring.cpp:23-52). mode "hash" (hashed priorities) or
    "ldf" (largest degree first). Changes the LU-SGS sweep order: a stated
    variant, not the reference's ordering."""
    m = {"hash": L.KF_COLOR_JP_HASH, "ldf": L.KF_COLOR_JP_LDF}[mode]
    nc, rounds = C.c_int(), C.c_int()
    _check(lib.kf_cloud_color_device(cloud.handle, device, m, seed, C.byref(nc), C.byref(rounds)))
    out = color_points(cloud)
    out.rounds = rounds.value
    return out


def order_wall_first(cloud: PointCloud) -> ColorAssignment:
    """The paper's Algorithm 5 sweep order: wall, interior
    and outer points swept as separate groups, each in its own colour order
    (levels (kind, colour), wall < interior < outer), built from the cloud's
    current colouring. A stated variant, not the reference's ordering."""
    _check(lib.kf_cloud_order_wall_first(cloud.handle, None))
    return color_points(cloud)


# ------------------------------------------------------------------ config
class SolverVariant(enum.IntEnum):
    Explicit = 0
    Anandh = 1
    AnandhAD = 2
    Manish = 3
    ManishAD = 4

    @classmethod
    def parse(cls, name: str) -> "SolverVariant":
        table = {"explicit": cls.Explicit, "anandh": cls.Anandh, "anandh_ad": cls.AnandhAD,
                 "manish": cls.Manish, "manish_ad": cls.ManishAD}
        if name not in table:
            raise ValueError(f"unknown variant '{name}'")
        return table[name]

    @property
    def label(self) -> str:
        return ["explicit", "anandh", "anandh_ad", "manish", "manish_ad"][int(self)]


class BcMode(enum.IntEnum):
    Physical = 0
    FreestreamAll = 1


@dataclass
class SolverConfig:
    """SolverConfig (driver.hpp:37-52) plus device options."""
    variant: SolverVariant = SolverVariant.Explicit
    cfl: float = 0.2
    n_iterations: int = 100
    n_inner: int = 3
    mach_inf: float = 0.63
    aoa_deg: float = 0.0
    convergence_decades: float = 0.0
    bc_mode: BcMode = BcMode.Physical
    cfl_ramp_iters: int = 0
    cfl_start: float = 0.0
    divergence_factor: float = 1e6
    device: int = 0
    ordering: int = 1       # in-colour point order: 0 natural, 1 Morton (default), 2 RCM
    use_graph: bool = True

    def to_c(self) -> L.Config:
        v = self.variant if not isinstance(self.variant, str) else SolverVariant.parse(self.variant)
        return L.Config(int(v), self.cfl, self.n_iterations, self.n_inner, self.mach_inf,
                        self.aoa_deg, self.convergence_decades, int(self.bc_mode),
                        self.cfl_ramp_iters, self.cfl_start, self.divergence_factor,
                        self.device, self.ordering, int(bool(self.use_graph)))


@dataclass
class IterationRecord:
    residual: float
    cl: float
    cd: float
    seconds: float
    counters: tuple
    sweep: tuple
    first_order_points: int


@dataclass
class RunHistory:
    iters: List[IterationRecord] = field(default_factory=list)
    diverged: bool = False
    abort_reason: str = ""
    loop_seconds: float = 0.0
    points: int = 0
    abort_point: int = -1
    final_state: Optional[np.ndarray] = None

    def iterations_to_decades(self, decades: float) -> int:
        """driver.cpp:169-178"""
        if not self.iters:
            return 0
        r0 = self.iters[0].residual
        if not (r0 > 0.0):
            return 1
        target = r0 * math.pow(10.0, -decades)
        for k, r in enumerate(self.iters):
            if r.residual <= target:
                return k + 1
        return 0

    @property
    def residual(self):
        return np.array([r.residual for r in self.iters])

    @property
    def cl(self):
        return np.array([r.cl for r in self.iters])

    @property
    def cd(self):
        return np.array([r.cd for r in self.iters])

    @property
    def first_order(self):
        return np.array([r.first_order_points for r in self.iters], np.int32)


def _records(buf, n):
    return [IterationRecord(r.residual, r.cl, r.cd, r.seconds, tuple(r.counters), tuple(r.sweep),
                            r.first_order_points) for r in buf[:n]]


# ------------------------------------------------------------------ solver
_PART_MODES = {"angular": L.KF_PART_ANGULAR, "morton": L.KF_PART_MORTON}


def _host_callbacks(exchange, allreduce):
    """ctypes trampolines for kf_exchange_fn / kf_allreduce_fn (a Python
    exception becomes a nonzero return: the library raises KF_RUNTIME)."""
    from . import _lib

    def exch(_user, n, peer, is_send, buf, nbytes):
        try:
            msgs = []
            for k in range(n):
                b = int(nbytes[k])
                arr = np.ctypeslib.as_array(C.cast(buf[k], C.POINTER(C.c_uint8)), shape=(b,))
                msgs.append((int(peer[k]), bool(is_send[k]), arr))
            exchange(msgs)
            return 0
        except Exception:  # pragma: no cover - reported as KF_RUNTIME
            import traceback
            traceback.print_exc()
            return 1

    def ared(_user, buf, n):
        try:
            allreduce(np.ctypeslib.as_array(buf, shape=(int(n),)))
            return 0
        except Exception:  # pragma: no cover
            import traceback
            traceback.print_exc()
            return 1

    return _lib.EXCHANGE_FN(exch), _lib.ALLREDUCE_FN(ared)


def _part_mode(mode) -> int:
    if isinstance(mode, str):
        if mode not in _PART_MODES:
            raise ValueError(f"unknown partition mode '{mode}'")
        return _PART_MODES[mode]
    return int(mode)


class Solver:
    """A device context (kf_ctx): one uploaded cloud + configuration.

    ``n_parts > 1`` splits the cloud into that many partitions held by this
    process on ``config.device`` (the domain-decomposed solver, halos
    refreshed by device copies); ``Solver.for_rank`` is the one-process-per-GPU
    form over NCCL.
    """

    def __init__(self, cloud: PointCloud, config: SolverConfig, n_parts: int = 1,
                 partition="angular", _rank=None):
        self.cloud = cloud
        self.config = config
        self.n = cloud.n()
        self._cfg = config.to_c()
        h = C.c_void_p()
        self._callbacks = None
        if _rank is not None and len(_rank) == 4:
            n_ranks, rank, exchange, allreduce = _rank
            self._callbacks = _host_callbacks(exchange, allreduce)  # kept alive with the context
            _check(lib.kf_create_rank_host(cloud.handle, C.byref(self._cfg), n_ranks, rank, _part_mode(partition),
                                           self._callbacks[0], self._callbacks[1], None, C.byref(h)))
        elif _rank is not None:
            n_ranks, rank, nccl_id = _rank
            _check(lib.kf_create_rank(cloud.handle, C.byref(self._cfg), n_ranks, rank, _part_mode(partition),
                                      nccl_id, C.byref(h)))
        elif n_parts == 1:
            _check(lib.kf_create(cloud.handle, C.byref(self._cfg), C.byref(h)))
        else:
            _check(lib.kf_create_partitioned(cloud.handle, C.byref(self._cfg), n_parts,
                                             _part_mode(partition), C.byref(h)))
        self._h = h

    @classmethod
    def for_rank(cls, cloud: PointCloud, config: SolverConfig, n_ranks: int, rank: int,
                 nccl_id: bytes, partition="angular") -> "Solver":
        """Partition `rank` of an `n_ranks`-way decomposition, one process per
        GPU; every rank passes the same cloud, config and NCCL id
        (``nccl_unique_id()`` on rank 0, broadcast by the caller). Host state
        arrays keep the whole-cloud shape; only this rank's owned entries are
        written."""
        return cls(cloud, config, partition=partition, _rank=(n_ranks, rank, nccl_id))

    @classmethod
    def for_rank_host(cls, cloud: PointCloud, config: SolverConfig, n_ranks: int, rank: int, exchange,
                      allreduce, partition="angular") -> "Solver":
        """Partition `rank` of an `n_ranks`-way decomposition over any host
        communicator (kf_create_rank_host): ``exchange(msgs)`` receives the
        step's posted messages as a list of ``(peer, is_send, buffer)`` with
        `buffer` a writable uint8 numpy view of pinned host memory, in
        posting order (the k-th send to a peer matches that peer's k-th
        receive), and must move them; ``allreduce(buf)`` sums a float64
        numpy array in place across the ranks. Launches are eager."""
        return cls(cloud, config, partition=partition, _rank=(n_ranks, rank, exchange, allreduce))

    @property
    def n_parts(self) -> int:
        return lib.kf_n_parts(self._h)

    @property
    def owned_points(self) -> int:
        return lib.kf_owned_points(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            lib.kf_destroy(h)
            self._h = None

    def close(self):
        self.__del__()

    # -- whole run -----------------------------------------------------------
    def run(self, want_state=True) -> RunHistory:
        cap = max(self.config.n_iterations, 1)
        recs = (L.IterRecord * cap)()
        nd = C.c_int()
        ls = C.c_double()
        fs = np.zeros((self.n, 4)) if want_state else None
        st = lib.kf_run(self._h, recs, C.byref(nd), _ptr(fs), C.byref(ls))
        h = RunHistory(_records(recs, nd.value), points=self.n, loop_seconds=ls.value,
                       final_state=fs)
        if st.code == L.KF_DIVERGED:
            h.diverged = True
            h.abort_reason = st.reason.decode()
            h.abort_point = st.point
        else:
            _check(st)
        return h

    # -- stepping --------------------------------------------------------------
    def reset(self):
        _check(lib.kf_reset(self._h))

    def set_state(self, U, dU_prev=None):
        d = None if dU_prev is None else _f64(dU_prev, (self.n, 4))
        _check(lib.kf_set_state(self._h, _f64(U, (self.n, 4)), _ptr(d)))

    def get_state(self, with_dU=False):
        U = np.zeros((self.n, 4))
        dU = np.zeros((self.n, 4)) if with_dU else None
        _check(lib.kf_get_state(self._h, U, _ptr(dU)))
        return (U, dU) if with_dU else U

    def iterate_async(self, n=1):
        _check(lib.kf_iterate_async(self._h, n))

    def sync_records(self, capacity=None):
        cap = capacity or max(self.config.n_iterations, 1)
        recs = (L.IterRecord * cap)()
        nd = C.c_int()
        st = lib.kf_sync_records(self._h, recs, cap, C.byref(nd))
        return _records(recs, min(nd.value, cap)), st

    def _out_f64(self, a, name):
        """A caller-supplied output must be a writable C-contiguous float64
        (n, 4) array: native code writes n*4 doubles through its pointer."""
        if a is None:
            return np.zeros((self.n, 4))
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.shape == (self.n, 4)
                and a.flags.c_contiguous and a.flags.writeable):
            raise ConfigError(f"{name} must be a writable C-contiguous float64 array of shape ({self.n}, 4)")
        return a

    def _in_f64(self, a, name):
        if a is None:
            raise ConfigError(f"{name} is required (pass zeros for the first iteration, driver.cpp:210)")
        a = _f64(a)
        if a.size != self.n * 4:
            raise ConfigError(f"{name} must hold {self.n} x 4 doubles, got {a.size}")
        return a.reshape(self.n, 4)

    def step_host(self, U_in, dU_prev_in, U_out=None, dU_out=None):
        U_in = self._in_f64(U_in, "U_in")
        dU_prev_in = self._in_f64(dU_prev_in, "dU_prev_in")
        U_out = self._out_f64(U_out, "U_out")
        if dU_out is not None:
            dU_out = self._out_f64(dU_out, "dU_out")
        rec = L.IterRecord()
        st = lib.kf_step_host(self._h, _ptr(U_in), _ptr(dU_prev_in), _ptr(U_out), _ptr(dU_out),
                              C.byref(rec))
        _check(st)
        return U_out, _records([rec], 1)[0]

    def _batch_ptrs(self, xs, name, out):
        """Raw pointers of a list of (n, 4) float64 buffers (numpy arrays or
        torch tensors, e.g. pinned host memory), validated like step_host's."""
        ptrs = []
        for k, x in enumerate(xs):
            if hasattr(x, "data_ptr"):  # torch tensor
                import torch
                ok = (x.dtype == torch.float64 and tuple(x.shape) == (self.n, 4) and x.is_contiguous()
                      and x.device.type == "cpu")
                if not ok:
                    raise ConfigError(f"{name}[{k}] must be a contiguous float64 CPU tensor of shape ({self.n}, 4)")
                ptrs.append(x.data_ptr())
            else:
                if out:
                    x = self._out_f64(x, f"{name}[{k}]")
                elif not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.shape == (self.n, 4)
                          and x.flags.c_contiguous):
                    raise ConfigError(f"{name}[{k}] must be a C-contiguous float64 array of shape ({self.n}, 4)")
                ptrs.append(x.ctypes.data)
        return ptrs

    def step_host_batch(self, U_in, dU_prev_in, U_out, dU_out=None):
        """len(U_in) independent host-fed steps, pipelined (kf_step_host_batch).
        Arguments are lists of (n, 4) float64 arrays (pinned for overlap);
        returns the records."""
        m = len(U_in)
        if len(dU_prev_in) != m or len(U_out) != m or (dU_out is not None and len(dU_out) != m):
            raise ConfigError("step_host_batch: every buffer list needs one entry per step")
        P = C.c_void_p * m
        pa = lambda ptrs: P(*ptrs)
        recs = (L.IterRecord * max(m, 1))()
        a_in = pa(self._batch_ptrs(U_in, "U_in", False))
        a_dprev = pa(self._batch_ptrs(dU_prev_in, "dU_prev_in", False))
        a_out = pa(self._batch_ptrs(U_out, "U_out", True))
        a_dout = None if dU_out is None else pa(self._batch_ptrs(dU_out, "dU_out", True))
        st = lib.kf_step_host_batch(self._h, m, a_in, a_dprev, a_out, a_dout, recs)
        _check(st)
        return _records(recs, m)

    def bench_mode(self, on=True):
        _check(lib.kf_bench_mode(self._h, int(bool(on))))

    @property
    def stream_ptr(self) -> int:
        return lib.kf_stream(self._h) or 0

    @property
    def launches_per_iteration(self) -> int:
        return lib.kf_launches_per_iteration(self._h)

    def profile_kernels(self, reps=3):
        """[(kernel name, mean ms per launch)] of one iteration, in launch order."""
        cap = 256
        names = C.create_string_buffer(32 * cap)
        ms = (C.c_float * cap)()
        n = C.c_int()
        _check(lib.kf_profile_kernels(self._h, reps, names, ms, cap, C.byref(n)))
        raw = names.raw
        return [(raw[32 * k:32 * k + 32].split(b"\0")[0].decode(), float(ms[k]))
                for k in range(min(n.value, cap))]

    # -- stage hooks ---------------------------------------------------------------
    def q(self, U):
        q = np.zeros((self.n, 4))
        _check(lib.kf_stage_q(self._h, _f64(U, (self.n, 4)), q))
        return q

    def grads(self, q):
        qx, qy = np.zeros((self.n, 4)), np.zeros((self.n, 4))
        _check(lib.kf_stage_grads(self._h, _f64(q, (self.n, 4)), qx, qy))
        return qx, qy

    def residual(self, q, qx, qy):
        R = np.zeros((self.n, 4))
        dem = np.zeros(self.n, np.int32)
        _check(lib.kf_stage_residual(self._h, _f64(q, (self.n, 4)), _f64(qx, (self.n, 4)),
                                     _f64(qy, (self.n, 4)), R, _ptr(dem)))
        return R, dem

    def lusgs(self, U, R, dU_prev, cfl):
        dt, d = np.zeros(self.n), np.zeros(self.n)
        S, dUs, dU = (np.zeros((self.n, 4)) for _ in range(3))
        _check(lib.kf_stage_lusgs(self._h, _f64(U, (self.n, 4)), _f64(R, (self.n, 4)),
                                  _f64(dU_prev, (self.n, 4)), cfl, _ptr(dt), _ptr(S), _ptr(d),
                                  _ptr(dUs), _ptr(dU)))
        return dict(dt=dt, S=S, diag=d, dU_star=dUs, dU=dU)

    def update(self, U, dU):
        out = np.zeros((self.n, 4))
        _check(lib.kf_stage_update(self._h, _f64(U, (self.n, 4)), _f64(dU, (self.n, 4)), out))
        return out

    def forces(self, U):
        cl, cd = C.c_double(), C.c_double()
        _check(lib.kf_stage_forces(self._h, _f64(U, (self.n, 4)), C.byref(cl), C.byref(cd)))
        return cl.value, cd.value


# ------------------------------------------------------ domain decomposition
def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0 of a multi-process run)."""
    buf = C.create_string_buffer(L.KF_NCCL_ID_BYTES)
    _check(lib.kf_nccl_unique_id(buf))
    return buf.raw


def partition_plan(cloud: PointCloud, n_parts: int, mode="angular") -> np.ndarray:
    """Owner partition of every point (kf_partition_plan)."""
    owner = np.zeros(cloud.n(), np.int32)
    _check(lib.kf_partition_plan(cloud.handle, n_parts, _part_mode(mode), owner))
    return owner


class LocalLayout:
    """Host-side local numbering and halo plan of one partition (kf_layout)."""

    def __init__(self, cloud: PointCloud, owner, n_parts: int, rank: int, ordering: int = 1):
        h = C.c_void_p()
        _check(lib.kf_layout_build(cloud.handle, np.ascontiguousarray(owner, np.int32), n_parts, rank,
                                   ordering, C.byref(h)))
        self._h = h
        a, b, c, d = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        lib.kf_layout_sizes(h, C.byref(a), C.byref(b), C.byref(c), C.byref(d))
        self.n_local, self.n_owned, self.n_colors, self.n_peers = a.value, b.value, c.value, d.value
        self.perm = np.zeros(self.n_local, np.int32)
        self.ghost = np.zeros(self.n_local, np.uint8)
        self.gs, self.oe, self.ge = (np.zeros(self.n_colors, np.int32) for _ in range(3))
        self.peers = np.zeros(max(self.n_peers, 1), np.int32)
        lib.kf_layout_arrays(h, _ptr(self.perm), _ptr(self.ghost), _ptr(self.gs), _ptr(self.oe),
                             _ptr(self.ge), _ptr(self.peers))
        self.peers = self.peers[:self.n_peers]
        self.ob = np.zeros(self.n_colors, np.int32)
        lib.kf_layout_boundary_end(h, _ptr(self.ob))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            lib.kf_layout_free(h)
            self._h = None

    def send(self, peer_slot: int, color: int) -> np.ndarray:
        m = lib.kf_layout_send(self._h, peer_slot, color, None)
        out = np.zeros(max(m, 0), np.int32)
        if m > 0:
            lib.kf_layout_send(self._h, peer_slot, color, _ptr(out))
        return out

    def recv(self, peer_slot: int, color: int):
        off = C.c_int()
        m = lib.kf_layout_recv(self._h, peer_slot, color, C.byref(off))
        return off.value, m


def run_fixed_point(cloud: PointCloud, config: SolverConfig, colors=None) -> RunHistory:
    """The drop-in seam (driver.hpp:101-106): B200 run of the fixed-point loop."""
    if colors is not None:
        if isinstance(colors, ColorAssignment):
            colors = colors.color
        elif isinstance(colors, SweepPlan):
            colors = colors.color_of
        set_colors(cloud, colors)
    s = Solver(cloud, config)
    try:
        return s.run()
    finally:
        s.close()


# ---------------------------------------------------------- point physics
def _probe(fn, U, *args):
    U = _f64(U).reshape(-1, 4)
    out = np.zeros_like(U)
    _check(fn(len(U), U, *args, out))
    return out


def split_flux(U, axis: int, sign: int):
    """Device split_flux(U, axis, sign) for a batch of states (kinetics.cpp:72-75)."""
    return _probe(lib.kf_probe_split_flux, U, axis, sign)


def jvp_split(U, dU, axis: int, sign: int, exact: bool = True):
    U = _f64(U).reshape(-1, 4)
    return _probe(lib.kf_probe_jvp_split, U, _f64(dU).reshape(-1, 4), axis, sign, int(exact))


def jvp_full(U, dU, axis: int, exact: bool = True):
    U = _f64(U).reshape(-1, 4)
    return _probe(lib.kf_probe_jvp_full, U, _f64(dU).reshape(-1, 4), axis, int(exact))


def measure_fp64_peak(device: int = 0) -> float:
    """Measured FP64 DFMA throughput in TFLOP/s (the FP64-pipe roofline)."""
    t = C.c_double()
    _check(lib.kf_measure_fp64_peak(device, C.byref(t)))
    return t.value


def device_count() -> int:
    return lib.kf_device_count()


def version() -> str:
    return lib.kf_version().decode()
