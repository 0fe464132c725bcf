"""ctypes binding of libspardl_cuda.so (the C ABI in include/spardl_cuda.h).

The library is built in-tree (paper_2304_00737_b200/libspardl_cuda.so) by
``__graft_entry__.build()`` / ``make -C paper_2304_00737_b200/csrc``.  There is
no fallback: if the library is missing, importing the device API raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libspardl_cuda.so")

# status codes <-> reference exception classes (inc/error.hpp:23-75)
STATUS = {
    1: "error",
    2: "partition_error",
    3: "block_mismatch_error",
    4: "schedule_violation_error",
    5: "theorem_violation_error",
    6: "group_size_error",
    7: "config_error",
    8: "state_error",
    9: "consistency_error",
    100: "cuda_error",
    101: "nccl_error",
    102: "argument_error",
    103: "unsupported_error",
}


class SpardlError(RuntimeError):
    """spardl::error (inc/error.hpp:23)."""

    kind = "error"

    def __init__(self, msg: str, code: int = 1):
        super().__init__(msg)
        self.code = code


def _sub(name, base=SpardlError):
    return type(name, (base,), {"kind": name})


PartitionError = _sub("partition_error")
BlockMismatchError = _sub("block_mismatch_error")
ScheduleViolationError = _sub("schedule_violation_error")
TheoremViolationError = _sub("theorem_violation_error")
GroupSizeError = _sub("group_size_error")
ConfigError = _sub("config_error")
StateError = _sub("state_error")
ConsistencyError = _sub("consistency_error")
CudaError = _sub("cuda_error")
NcclError = _sub("nccl_error")
ArgumentError = _sub("argument_error")
UnsupportedError = _sub("unsupported_error")

_BY_CODE = {
    1: SpardlError,
    2: PartitionError,
    3: BlockMismatchError,
    4: ScheduleViolationError,
    5: TheoremViolationError,
    6: GroupSizeError,
    7: ConfigError,
    8: StateError,
    9: ConsistencyError,
    100: CudaError,
    101: NcclError,
    102: ArgumentError,
    103: UnsupportedError,
}


class Config(C.Structure):
    """spardl_config == spardl::ClusterConfig (inc/pipeline.hpp:39-52)."""

    _fields_ = [
        ("workers", C.c_int64),
        ("dimension", C.c_int64),
        ("k", C.c_int64),
        ("teams", C.c_int64),
        ("sag", C.c_int32),
        ("residual", C.c_int32),
        ("timing", C.c_int32),
        ("pad_", C.c_int32),
        ("seed", C.c_uint64),
    ]


class RunInfo(C.Structure):
    _fields_ = [
        ("consistent", C.c_int32),
        ("conservation_applicable", C.c_int32),
        ("conservation_error", C.c_double),
        ("max_rounds", C.c_int64),
        ("max_scalars", C.c_int64),
        ("srs_rounds", C.c_int64),
        ("srs_scalars", C.c_int64),
        ("sag_rounds", C.c_int64),
        ("sag_scalars", C.c_int64),
        ("gather_rounds", C.c_int64),
        ("gather_scalars", C.c_int64),
        ("pred_rounds", C.c_int64),
        ("pred_low", C.c_int64),
        ("pred_high", C.c_int64),
        ("n_union", C.c_int64),
        ("global_nnz", C.c_int64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class HCtrl(C.Structure):
    _fields_ = [
        ("lower", C.c_double),
        ("upper", C.c_double),
        ("target", C.c_int64),
        ("h", C.c_double),
        ("step", C.c_double),
        ("flag", C.c_int32),
        ("pad_", C.c_int32),
    ]


# every symbol include/spardl_cuda.h declares (tests check the exports)
EXPORTS = [
    "spardl_last_error", "spardl_device_count", "spardl_abi_version", "spardl_validate", "spardl_partition",
    "spardl_block_of", "spardl_build_bags", "spardl_expected_cost_srs",
    "spardl_expected_cost_sag", "spardl_bsag_phase_cost", "spardl_topka_cost",
    "spardl_dyadic_shares", "spardl_hctrl_init", "spardl_hctrl_observe", "spardl_hctrl_budget",
    "spardl_topk_select", "spardl_topk_select_slice", "spardl_merge_add",
    "spardl_topk_select_f64", "spardl_merge_add_f64", "spardl_topk_select_f64_hostbuf",
    "spardl_merge_add_f64_hostbuf", "spardl_topk_select_hostbuf", "spardl_topk_select_slice_hostbuf", "spardl_merge_add_hostbuf",
    "spardl_nccl_unique_id", "spardl_ctx_create", "spardl_ctx_destroy", "spardl_plan_ops",
    "spardl_ctx_local_workers", "spardl_ctx_set_graph", "spardl_ctx_set_audit",
    "spardl_allreduce", "spardl_allreduce_host", "spardl_profile", "spardl_sync",
    "spardl_get_run_info", "spardl_get_global", "spardl_get_carry", "spardl_ctx_reset_state",
    "spardl_carry_to_host", "spardl_carry_from_host", "spardl_set_controller",
    "spardl_get_ledger", "spardl_get_union_sizes", "spardl_get_controller",
    "spardl_dense_fallbacks", "spardl_dense_fallbacks_total", "spardl_wide_handed_back", "spardl_candidate_retries", "spardl_div_diag", "spardl_kernel_launches", "spardl_ctx_stream",
    "spardl_ctx_transport", "spardl_debug_select_timestamps", "spardl_mctx_create",
    "spardl_mctx_destroy", "spardl_mctx_devices", "spardl_mctx_allreduce",
    "spardl_mctx_allreduce_host", "spardl_mctx_sync", "spardl_mctx_get_run_info",
    "spardl_mctx_get_ledger", "spardl_mctx_get_union_sizes", "spardl_mctx_get_global",
    "spardl_mctx_carry_to_host", "spardl_mctx_carry_from_host", "spardl_mctx_set_controller",
    "spardl_mctx_get_controller", "spardl_mctx_reset_state",
]

_lib = None


def lib() -> C.CDLL:
    """Load libspardl_cuda.so (raises if it was not built: no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (the SparDL device path has no CPU fallback)")
    try:
        # torch bundles a newer libnccl.so.2; load it first so the soname
        # resolves to the same library for torch and for us
        import torch  # noqa: F401
    except ImportError:
        pass
    L = C.CDLL(LIB_PATH)
    L.spardl_last_error.restype = C.c_char_p
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().spardl_last_error().decode()
        raise _BY_CODE.get(rc, SpardlError)(msg, rc)
