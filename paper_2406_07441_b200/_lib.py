"""ctypes binding of libkf.so (include/kf.h).

The shared library is built in-tree by ``make -C paper_2406_07441_b200/csrc``
(``__graft_entry__.build()``). There is no fallback: if the library is
missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# KF_LIB_PATH: an alternative in-tree build (A/B experiments of build flags)
LIB_PATH = os.environ.get("KF_LIB_PATH") or os.path.join(HERE, "libkf.so")

KF_OK, KF_INVALID_STATE, KF_INVALID_INCREMENT, KF_DIVERGED, KF_CONFIG, KF_CUDA, KF_RUNTIME = range(7)

# every symbol include/kf.h declares (tests/test_abi.py checks the export list)
EXPORTED = [
    "kf_cloud_generate_naca", "kf_cloud_load", "kf_cloud_save", "kf_cloud_save_binary", "kf_cloud_from_arrays",
    "kf_cloud_free", "kf_cloud_n", "kf_cloud_n_colors", "kf_cloud_set_colors",
    "kf_cloud_geometry", "kf_cloud_list_nnz", "kf_cloud_list", "kf_cloud_ls_full",
    "kf_cloud_ls_split", "kf_cloud_flagged", "kf_cloud_colors", "kf_cloud_report",
    "kf_config_default", "kf_create", "kf_destroy", "kf_run", "kf_reset", "kf_set_state",
    "kf_get_state", "kf_iterate_async", "kf_sync_records", "kf_step_host", "kf_bench_mode",
    "kf_stream", "kf_launches_per_iteration", "kf_stage_q", "kf_stage_grads",
    "kf_stage_residual", "kf_stage_lusgs", "kf_stage_update", "kf_stage_forces",
    "kf_probe_split_flux", "kf_probe_jvp_split", "kf_probe_jvp_full", "kf_version",
    "kf_device_count", "kf_profile_kernels", "kf_measure_fp64_peak",
    "kf_partition_plan", "kf_layout_build", "kf_layout_free", "kf_layout_sizes",
    "kf_layout_arrays", "kf_layout_send", "kf_layout_recv", "kf_create_partitioned",
    "kf_nccl_unique_id", "kf_create_rank", "kf_create_rank_host", "kf_n_parts", "kf_owned_points", "kf_step_host_batch",
    "kf_probe_math", "kf_cloud_color_device", "kf_cloud_order_wall_first", "kf_layout_boundary_end",
]

KF_NCCL_ID_BYTES = 128
KF_PART_ANGULAR, KF_PART_MORTON = 0, 1
KF_COLOR_JP_HASH, KF_COLOR_JP_LDF = 0, 1


class Status(C.Structure):
    _fields_ = [("code", C.c_int), ("point", C.c_int), ("iteration", C.c_int),
                ("reason", C.c_char * 192)]


class Config(C.Structure):
    _fields_ = [
        ("variant", C.c_int), ("cfl", C.c_double), ("n_iterations", C.c_int),
        ("n_inner", C.c_int), ("mach_inf", C.c_double), ("aoa_deg", C.c_double),
        ("convergence_decades", C.c_double), ("bc_mode", C.c_int),
        ("cfl_ramp_iters", C.c_int), ("cfl_start", C.c_double),
        ("divergence_factor", C.c_double), ("device", C.c_int), ("ordering", C.c_int),
        ("use_graph", C.c_int),
    ]


class IterRecord(C.Structure):
    _fields_ = [
        ("residual", C.c_double), ("cl", C.c_double), ("cd", C.c_double),
        ("seconds", C.c_double), ("counters", C.c_uint64 * 5), ("sweep", C.c_uint64 * 5),
        ("first_order_points", C.c_int),
    ]


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_S = Status
_pp = C.POINTER(C.c_void_p)
# kf_exchange_fn / kf_allreduce_fn (include/kf.h, host-staged transport)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                          C.POINTER(C.c_void_p), C.POINTER(C.c_size_t))
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_size_t)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2406_07441_b200/csrc` "
            "(or __graft_entry__.build()). The B200 path has no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    sig = {
        "kf_cloud_generate_naca": (_S, [C.c_char_p, C.c_int, C.c_int, C.c_double, _pp]),
        "kf_cloud_load": (_S, [C.c_char_p, _pp]),
        "kf_cloud_save": (_S, [_vp, C.c_char_p]),
        "kf_cloud_save_binary": (_S, [_vp, C.c_char_p]),
        "kf_cloud_from_arrays": (_S, [C.c_int, _dp, _dp, _ip, _dp, _dp, _ip, _ip, _pp]),
        "kf_cloud_free": (None, [_vp]),
        "kf_cloud_n": (C.c_int, [_vp]),
        "kf_cloud_n_colors": (C.c_int, [_vp]),
        "kf_cloud_set_colors": (_S, [_vp, _ip]),
        "kf_cloud_color_device": (_S, [_vp, C.c_int, C.c_int, C.c_uint, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "kf_cloud_order_wall_first": (_S, [_vp, C.POINTER(C.c_int)]),
        "kf_cloud_geometry": (None, [_vp, _dp, _dp, _ip, _dp, _dp]),
        "kf_cloud_list_nnz": (C.c_long, [_vp, C.c_int]),
        "kf_cloud_list": (None, [_vp, C.c_int, _ip, _ip]),
        "kf_cloud_ls_full": (None, [_vp, _dp, _dp, _ip]),
        "kf_cloud_ls_split": (None, [_vp, C.c_int, _dp, _dp, _ip]),
        "kf_cloud_flagged": (C.c_int, [_vp, _vp]),
        "kf_cloud_colors": (None, [_vp, _ip]),
        "kf_cloud_report": (None, [_vp, _vp, C.POINTER(C.c_int), _vp, C.POINTER(C.c_int)]),
        "kf_config_default": (None, [C.POINTER(Config)]),
        "kf_create": (_S, [_vp, C.POINTER(Config), _pp]),
        "kf_destroy": (None, [_vp]),
        "kf_run": (_S, [_vp, _vp, C.POINTER(C.c_int), _vp, C.POINTER(C.c_double)]),
        "kf_reset": (_S, [_vp]),
        "kf_set_state": (_S, [_vp, _dp, _vp]),
        "kf_get_state": (_S, [_vp, _dp, _vp]),
        "kf_iterate_async": (_S, [_vp, C.c_int]),
        "kf_sync_records": (_S, [_vp, _vp, C.c_int, C.POINTER(C.c_int)]),
        "kf_step_host": (_S, [_vp, _vp, _vp, _vp, _vp, _vp]),
        "kf_bench_mode": (_S, [_vp, C.c_int]),
        "kf_step_host_batch": (_S, [_vp, C.c_int, _vp, _vp, _vp, _vp, _vp]),
        "kf_stream": (_vp, [_vp]),
        "kf_launches_per_iteration": (C.c_int, [_vp]),
        "kf_stage_q": (_S, [_vp, _dp, _dp]),
        "kf_stage_grads": (_S, [_vp, _dp, _dp, _dp]),
        "kf_stage_residual": (_S, [_vp, _dp, _dp, _dp, _dp, _vp]),
        "kf_stage_lusgs": (_S, [_vp, _dp, _dp, _dp, C.c_double, _vp, _vp, _vp, _vp, _vp]),
        "kf_stage_update": (_S, [_vp, _dp, _dp, _dp]),
        "kf_stage_forces": (_S, [_vp, _dp, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "kf_probe_split_flux": (_S, [C.c_int, _dp, C.c_int, C.c_int, _dp]),
        "kf_probe_math": (_S, [C.c_int, C.c_int, _dp, _dp, _dp]),
        "kf_probe_jvp_split": (_S, [C.c_int, _dp, _dp, C.c_int, C.c_int, C.c_int, _dp]),
        "kf_probe_jvp_full": (_S, [C.c_int, _dp, _dp, C.c_int, C.c_int, _dp]),
        "kf_profile_kernels": (_S, [_vp, C.c_int, C.c_char_p, _vp, C.c_int, C.POINTER(C.c_int)]),
        "kf_measure_fp64_peak": (_S, [C.c_int, C.POINTER(C.c_double)]),
        "kf_partition_plan": (_S, [_vp, C.c_int, C.c_int, _ip]),
        "kf_layout_build": (_S, [_vp, _ip, C.c_int, C.c_int, C.c_int, _pp]),
        "kf_layout_free": (None, [_vp]),
        "kf_layout_sizes": (None, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_int)]),
        "kf_layout_arrays": (None, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
        "kf_layout_boundary_end": (None, [_vp, _vp]),
        "kf_layout_send": (C.c_int, [_vp, C.c_int, C.c_int, _vp]),
        "kf_layout_recv": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(C.c_int)]),
        "kf_create_partitioned": (_S, [_vp, C.POINTER(Config), C.c_int, C.c_int, _pp]),
        "kf_nccl_unique_id": (_S, [C.c_char_p]),
        "kf_create_rank": (_S, [_vp, C.POINTER(Config), C.c_int, C.c_int, C.c_int, C.c_char_p, _pp]),
        "kf_create_rank_host": (_S, [_vp, C.POINTER(Config), C.c_int, C.c_int, C.c_int, EXCHANGE_FN,
                                     ALLREDUCE_FN, _vp, _pp]),
        "kf_n_parts": (C.c_int, [_vp]),
        "kf_owned_points": (C.c_int, [_vp]),
        "kf_version": (C.c_char_p, []),
        "kf_device_count": (C.c_int, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()
