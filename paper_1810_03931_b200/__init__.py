"""odegpu — B200-native ensemble ODE solver (hot path of arXiv 1810.03931).

The compute path is libodegpu.so (hand-written sm_100a CUDA behind the C ABI
in include/odegpu.h). This package is the thin host mirror used by tests and
bench.py; the C++ host API lives in include/odegpu/.
"""
from . import abi, models, scan, workloads  # noqa: F401
from .api import (  # noqa: F401
    BatchDims,
    CopyMode,
    DevicePool,
    InvalidArgument,
    LinearCopySpec,
    OdegpuError,
    OutOfRange,
    Pipeline,
    Unsupported,
    pinned,
    PoolDims,
    ProblemPool,
    RandomCopySpec,
    SolverBatch,
    SolverConfig,
    dfma_peak,
    flat_index,
    linear_set,
    linear_set_device,
    make_batch_dims,
    random_set,
    random_set_device,
    solve,
    solve_iteratively,
    batch_copy,
    slice_range,
    solve_pool,
)
