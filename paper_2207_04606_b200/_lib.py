"""ctypes binding of libstrata_b200.so (the C ABI declared in include/strata_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_2207_04606_b200/csrc``).  There is no fallback: if the library is missing, importing
this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# STRATA_B200_LIB: development override to A/B two in-tree builds of the same library.
LIB_PATH = os.environ.get("STRATA_B200_LIB") or os.path.join(_HERE, "libstrata_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first "
        "(python -c 'import __graft_entry__ as g; g.build()')")

lib = C.CDLL(LIB_PATH)

# Reference ErrKind (include/strata/common.hpp:36-45); code = ordinal + 1.
ERR_KINDS = {1: "Validation", 2: "Schedule", 3: "Lowering", 4: "Capacity", 5: "Lookup",
             6: "Usage", 7: "Exec", 8: "Internal", 9: "Cuda"}


class StrataError(RuntimeError):
    """Mirror of strata::Error{ErrKind kind, what()} (common.hpp:47-53)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.kind = ERR_KINDS.get(code, "Internal")


def check(rc: int) -> None:
    if rc != 0:
        raise StrataError(rc, lib.strata_last_error().decode())


i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f32p = C.POINTER(C.c_float)
vp = C.c_void_p
i64 = C.c_int64


def _sig(name, restype, *args):
    if os.environ.get("STRATA_B200_LIB") and not hasattr(lib, name):
        return None  # A/B against an older build: symbols it predates stay unbound
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = list(args)
    return fn


_sig("strata_last_error", C.c_char_p)
_sig("strata_abi_version", C.c_int)
_sig("strata_device_ok", C.c_int)
_sig("strata_generate_csr", C.c_int, C.c_char_p, i64, i64, C.c_double, i64, i64, C.c_double,
     C.c_uint64, C.POINTER(vp))
_sig("strata_csr_host_info", C.c_int, vp, i64p, i64p, i64p)
_sig("strata_csr_host_indptr", vp, vp)
_sig("strata_csr_host_indices", vp, vp)
_sig("strata_csr_host_values", vp, vp)
_sig("strata_csr_host_destroy", C.c_int, vp)
_sig("strata_csr_host_row_order", C.c_int, vp, vp)
_sig("strata_dense_int", C.c_int, i64, C.c_uint64, vp)
_sig("strata_hyb_decompose", C.c_int, vp, vp, vp, i64, i64, i64, C.c_int, C.c_int, vp,
     C.POINTER(vp))
_sig("strata_hyb_auto_k", C.c_int, i64, i64)
_sig("strata_hyb_num_parts", C.c_int, vp, C.POINTER(C.c_int))
_sig("strata_hyb_part_info", C.c_int, vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
     i64p, i64p, i64p, i64p, i64p, i64p)
_sig("strata_hyb_part_read", C.c_int, vp, C.c_int, vp, vp, vp, vp)
_sig("strata_hyb_get_part", C.c_int, vp, C.c_int, vp, vp, vp, vp, vp, vp, vp, vp)
_sig("strata_hyb_part_device", C.c_int, vp, C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp))
_sig("strata_hyb_padding_ratio", C.c_int, vp, C.POINTER(C.c_double))
_sig("strata_hyb_dims", C.c_int, vp, i64p, i64p, C.POINTER(C.c_int), C.POINTER(C.c_int))
_sig("strata_hyb_destroy", C.c_int, vp)
_sig("strata_hyb_schedule_info", C.c_int, vp, i64p, i64p, i64p, i64p, C.POINTER(C.c_int))
_sig("strata_hyb_row_work_balance", C.c_int, vp, C.POINTER(C.c_double), vp)
_sig("strata_gemm_f32", C.c_int, vp, vp, vp, i64, i64, i64, vp)
_sig("strata_gnn_layer_work_floats", i64, vp, i64, i64)
_sig("strata_gnn_layer_f32", C.c_int, vp, vp, vp, vp, vp, i64, i64, vp)
_sig("strata_spmm_hyb_f32", C.c_int, vp, vp, vp, i64, vp)
_sig("strata_spmm_hyb_f32_host", C.c_int, vp, vp, vp, i64, vp)
_sig("strata_spmm_hyb_f32_host_batch", C.c_int, vp, vp, vp, i64, i64, vp)
_sig("strata_spmm_hyb_f32_multi", C.c_int, vp, vp, vp, C.c_int, i64, vp)
_sig("strata_ipc_get_handle", C.c_int, vp, vp, i64p)
_sig("strata_ipc_open_handle", C.c_int, vp, C.POINTER(vp))
_sig("strata_ipc_close", C.c_int, vp)
_sig("strata_spmm_csr_f32", C.c_int, vp, vp, vp, vp, vp, i64, i64, i64, vp)
_sig("strata_sddmm_csr_f32", C.c_int, vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, vp)
_sig("strata_bsr_from_csr", C.c_int, vp, vp, vp, i64, i64, i64, i64, vp, C.POINTER(vp))
_sig("strata_bsr_info", C.c_int, vp, i64p, i64p, i64p, i64p, i64p)
_sig("strata_bsr_read", C.c_int, vp, vp, vp, vp)
_sig("strata_bsr_destroy", C.c_int, vp)
_sig("strata_bsr_spmm_bf16", C.c_int, vp, vp, vp, i64, vp)
_sig("strata_bsr_spmm_bf16_batched", C.c_int, vp, vp, vp, vp, i64, i64, vp)
_sig("strata_bsr_sddmm_bf16", C.c_int, vp, vp, vp, vp, i64, i64, vp)
_sig("strata_dbsr_from_csr", C.c_int, vp, vp, vp, i64, i64, i64, i64, vp, C.POINTER(vp))
_sig("strata_dbsr_info", C.c_int, vp, i64p, i64p, i64p, i64p, i64p, i64p)
_sig("strata_dbsr_read", C.c_int, vp, vp, vp, vp, vp)
_sig("strata_dbsr_destroy", C.c_int, vp)
_sig("strata_dbsr_spmm_bf16", C.c_int, vp, vp, vp, i64, vp)
_sig("strata_srbcrs_from_csr", C.c_int, vp, vp, vp, i64, i64, i64, i64, i64, vp, C.POINTER(vp))
_sig("strata_srbcrs_info", C.c_int, vp, i64p, i64p, i64p, i64p, i64p)
_sig("strata_srbcrs_read", C.c_int, vp, vp, vp, vp)
_sig("strata_srbcrs_destroy", C.c_int, vp)
_sig("strata_srbcrs_spmm_bf16", C.c_int, vp, vp, vp, i64, vp)
_sig("strata_attn_plan_create", C.c_int, vp, i64, i64, C.POINTER(vp), vp)
_sig("strata_attn_plan_destroy", C.c_int, vp)
_sig("strata_attn_csr_f32", C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, i64, vp)
_sig("strata_csr_from_coo", C.c_int, vp, vp, vp, i64, i64, i64, vp, vp, vp, vp)
_sig("strata_ell_from_csr", C.c_int, vp, vp, vp, i64, i64, i64, vp, vp, vp)
_sig("strata_rgms_bf16", C.c_int, vp, vp, vp, vp, i64, i64, i64, i64, vp, vp, vp, i64, i64, vp)
_sig("strata_rgms_plan", C.c_int, vp, vp, vp, vp, i64, i64, i64, i64, C.POINTER(vp), vp)
_sig("strata_rgms_run_bf16", C.c_int, vp, vp, vp, vp, i64, i64, vp)
_sig("strata_rgms_info", C.c_int, vp, i64p, i64p)
_sig("strata_rgms_destroy", C.c_int, vp)
_sig("strata_rgms_plan_hyb", C.c_int, vp, i64, C.POINTER(vp), vp)
_sig("strata_rgms_hyb_bf16", C.c_int, vp, i64, vp, vp, vp, i64, i64, vp)
_sig("strata_partition_rows", C.c_int, vp, i64, C.c_int, vp)
_sig("strata_nccl_unique_id", C.c_int, vp)
_sig("strata_nccl_comm_init", C.c_int, vp, C.c_int, C.c_int, vp)
_sig("strata_nccl_comm_destroy", C.c_int, vp)
_sig("strata_shard_plan_create", C.c_int, vp, vp, vp, i64, i64, C.c_int, C.c_int, C.c_int,
     C.c_int, C.c_int, C.POINTER(vp), vp)
_sig("strata_shard_plan_rows", C.c_int, vp, C.c_int, C.c_int, i64p, i64p)
_sig("strata_shard_plan_destroy", C.c_int, vp)
_sig("strata_spmm_hyb_f32_sharded", C.c_int, vp, vp, vp, i64, vp, C.c_int, vp)
_sig("strata_spmm_hyb_f32_sharded_p2p", C.c_int, vp, vp, vp, C.c_int, i64, vp)
_sig("strata_sddmm_csr_f32_sharded", C.c_int, vp, vp, vp, vp, i64, C.c_int, vp, C.c_int, vp)
_sig("strata_mtx_parse", C.c_int, vp, i64, C.POINTER(vp), vp)
_sig("strata_mtx_read_file", C.c_int, C.c_char_p, C.POINTER(vp), vp)
_sig("strata_mtx_info", C.c_int, vp, i64p, i64p, i64p)
_sig("strata_mtx_device", C.c_int, vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp))
_sig("strata_mtx_read", C.c_int, vp, vp, vp, vp)
_sig("strata_mtx_destroy", C.c_int, vp)

# Every symbol include/strata_b200.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "strata_last_error", "strata_abi_version", "strata_device_ok", "strata_generate_csr",
    "strata_csr_host_info", "strata_csr_host_indptr", "strata_csr_host_indices",
    "strata_csr_host_values", "strata_csr_host_destroy", "strata_csr_host_row_order",
    "strata_dense_int",
    "strata_hyb_decompose", "strata_hyb_auto_k", "strata_hyb_num_parts", "strata_hyb_part_info",
    "strata_hyb_part_read", "strata_hyb_get_part", "strata_hyb_part_device", "strata_hyb_padding_ratio",
    "strata_hyb_dims", "strata_hyb_destroy", "strata_hyb_schedule_info",
    "strata_hyb_row_work_balance", "strata_spmm_hyb_f32", "strata_spmm_hyb_f32_host",
    "strata_spmm_hyb_f32_host_batch", "strata_spmm_hyb_f32_multi", "strata_gnn_layer_work_floats",
    "strata_gnn_layer_f32", "strata_gemm_f32", "strata_ipc_get_handle",
    "strata_ipc_open_handle", "strata_ipc_close",
    "strata_spmm_csr_f32", "strata_sddmm_csr_f32", "strata_bsr_from_csr", "strata_bsr_info",
    "strata_bsr_read", "strata_bsr_destroy", "strata_bsr_spmm_bf16",
    "strata_bsr_spmm_bf16_batched", "strata_csr_from_coo",
    "strata_bsr_sddmm_bf16", "strata_dbsr_from_csr", "strata_dbsr_info", "strata_dbsr_read", "strata_dbsr_destroy",
    "strata_dbsr_spmm_bf16", "strata_srbcrs_from_csr", "strata_srbcrs_info", "strata_srbcrs_read",
    "strata_srbcrs_destroy", "strata_srbcrs_spmm_bf16", "strata_attn_plan_create",
    "strata_attn_plan_destroy", "strata_attn_csr_f32", "strata_ell_from_csr",
    "strata_rgms_bf16", "strata_rgms_plan", "strata_rgms_run_bf16", "strata_rgms_info",
    "strata_rgms_destroy", "strata_partition_rows", "strata_rgms_plan_hyb", "strata_rgms_hyb_bf16",
    "strata_mtx_parse", "strata_mtx_read_file", "strata_mtx_info", "strata_mtx_device",
    "strata_mtx_read", "strata_mtx_destroy",
    "strata_nccl_unique_id", "strata_nccl_comm_init", "strata_nccl_comm_destroy",
    "strata_shard_plan_create", "strata_shard_plan_rows", "strata_shard_plan_destroy",
    "strata_spmm_hyb_f32_sharded", "strata_spmm_hyb_f32_sharded_p2p",
    "strata_sddmm_csr_f32_sharded",
]
