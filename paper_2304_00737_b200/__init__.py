"""B200-native SparDL sparse gradient synchronisation (arXiv 2304.00737).

The hot path -- spardl_all_reduce of the reference
(/root/reference/proj/include/spardl/pipeline.hpp:140) -- runs in
libspardl_cuda.so (hand-written sm_100a CUDA + NCCL over NVLink), reached
through the C ABI in include/spardl_cuda.h.  This package is the Python view
of that ABI; it has no CPU implementation of the path.
"""
from ._lib import (  # noqa: F401
    ArgumentError, BlockMismatchError, ConfigError, ConsistencyError, CudaError, GroupSizeError,
    NcclError, PartitionError, ScheduleViolationError, SpardlError, StateError,
    TheoremViolationError, UnsupportedError, LIB_PATH, lib)
from .api import (  # noqa: F401
    BlockPartition, ClusterConfig, HController, SparDL, SparDLMulti, build_bags, bsag_phase_cost,
    dyadic_shares, expected_cost_sag, expected_cost_srs, merge_add, partition, top_k_select,
    top_k_select_slice, topka_cost, validate)
