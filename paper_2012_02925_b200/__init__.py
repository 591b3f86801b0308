"""B200-native drop-in for the multi-block finite-volume hot path of
arxiv 2012.02925 (reference: the `blockflow` package).

Public API (mirrors blockflow's stepping seam):

    iterate_gpu, run_distributed_gpu, GpuRankStepper, GpuContext
    IterationResult, DistributedResult, check_history_guards, write_residual_csv

Host-side setup mirrors (geometry, planning, topology, model, mms) let the
path run where the reference is not installed.  All arithmetic of the hot
path runs in libbfgpu.so (CUDA, sm_100a); there is no CPU fallback.
"""

from .errors import (BlockflowError, ConfigError, DivergenceError, NativeLibraryError,  # noqa: F401
                     NonPhysicalStateError)
from .model import FreestreamState, GasModel, SchemeConfig  # noqa: F401

__all__ = ["iterate_gpu", "run_distributed_gpu", "GpuRankStepper", "GpuContext",
           "IterationResult", "DistributedResult", "GasModel", "SchemeConfig",
           "FreestreamState"]


def __getattr__(name):
    # stepper pulls in ctypes/native lazily so that host-only users (planning,
    # tests of the mirrors) do not need the shared library.
    if name in ("iterate_gpu", "run_distributed_gpu", "GpuRankStepper", "GpuContext",
                "IterationResult", "DistributedResult", "check_history_guards",
                "write_residual_csv", "GpuBlockView"):
        from . import stepper
        return getattr(stepper, name)
    raise AttributeError(name)
