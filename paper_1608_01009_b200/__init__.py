"""B200-native fp64 particle-in-cell step (arXiv 1608.01009 hot path).

The product is libpic.so (CUDA, sm_100a) behind the C ABI in include/pic.h;
this package is its thin ctypes binding.  No oracle import, no CPU fallback.
"""
from .pic import (  # noqa: F401
    BC_OPEN, BC_PERIODIC, EXPORTS, balance_slabs, FLAG_LOCAL_GROUP, FLAG_NAIVE, FLAG_NO_GRAPH, FLAG_PROFILE, PicConfig, PicDiag, PicError,
    Simulation, broadcast_nccl_id, diagnostics_group, lib, make_config, nccl_unique_id, simulation_from_workload,
    step_group, workload_config,
)
