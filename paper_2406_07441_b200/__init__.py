"""kinfree-b200: B200-native (sm_100a, FP64) implicit-LSKUM hot path.

Drop-in for the reference kinfree solver's ``run_fixed_point``
(/root/reference/proj/include/kinfree/driver.hpp:101-106). The compute lives
in ``libkf.so`` (CUDA kernels + C++ host, C ABI in include/kf.h); this package
is the Python mirror of the reference API over that ABI.
"""
from .api import (  # noqa: F401
    BcMode,
    ColorAssignment,
    ConfigError,
    CudaError,
    InvalidIncrementError,
    InvalidStateError,
    IterationRecord,
    KinfreeError,
    LocalLayout,
    LsCoefficients,
    PointCloud,
    PointKind,
    RunHistory,
    Solver,
    SolverConfig,
    SolverVariant,
    SweepPlan,
    build_ls_coefficients,
    build_sweep_plan,
    color_points,
    color_points_device,
    device_count,
    generate_naca_ogrid,
    jvp_full,
    jvp_split,
    load_cloud,
    measure_fp64_peak,
    nccl_unique_id,
    order_wall_first,
    partition_plan,
    run_fixed_point,
    save_cloud,
    set_colors,
    split_flux,
    version,
)
from ._lib import LIB_PATH  # noqa: F401
