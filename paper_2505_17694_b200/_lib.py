"""ctypes binding of the C ABI declared in include/codec_b200.h.

The shared library `_codec_b200.so` (built in-tree by
`python -m paper_2505_17694_b200.build` / `__graft_entry__.build()`) is
the only implementation of the hot path: there is no Python or CPU
fallback. If the library is missing, every entry point raises
`LibraryNotBuilt` -- loudly, at the first call.

Status codes returned by the library are turned into the reference's
exception classes (errors.py) carrying the library's message.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import errors as E

LIB_PATH = Path(os.environ.get("CODEC_B200_LIB", Path(__file__).resolve().parent / "_codec_b200.so"))


class LibraryNotBuilt(RuntimeError):
    pass


_STATUS = {
    1: E.CycleDetected,
    2: E.DanglingParent,
    3: E.PathNotPrefixChain,
    4: E.DimensionMismatch,
    5: E.UnknownRequest,
    6: E.UnknownNode,
    7: E.ShapeMismatch,
    8: E.EmptyVisibleSet,
    9: E.NoVisibleTokens,
    10: E.PlanForestMismatch,
    11: E.IncompletePartials,
    12: E.SearchSpaceOverflow,
    13: E.ProfileLoadError,
    14: E.IncompleteGrid,
    15: E.NonPositiveCost,
    16: E.DuplicateKnot,
    20: ValueError,
    30: E.UnsupportedShape,
    31: E.CudaError,
}

P = C.c_void_p
I32, I64, F64 = C.c_int32, C.c_int64, C.c_double
PI32, PI64, PF64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_double)


class CostTableC(C.Structure):
    _fields_ = [("n_nq", I32), ("n_n", I32), ("nq_knots", PI64), ("n_knots", PI64), ("cost_ms", PF64)]


class IndexInfo(C.Structure):
    _fields_ = [("n_nodes", I32), ("bs", I32), ("total_tokens", I64), ("qset_nnz", I64), ("path_nnz", I64)]


class PlanInfo(C.Structure):
    _fields_ = [("n_tasks", I32), ("n_subtasks", I32), ("blocks", I32), ("truncated", I32),
                ("makespan_ms", F64), ("cost_l_ms", F64)]


class Dims(C.Structure):
    _fields_ = [("bs", I32), ("h_q", I32), ("h_kv", I32), ("d", I32), ("head_begin", I32),
                ("head_end", I32), ("kv_dtype", I32), ("flags", I32), ("pool_tokens", I64),
                ("sm_count", I32), ("tc_sm_budget", I32), ("page_size", I32), ("reserved0", I32),
                ("page_table", C.c_void_p)]


class TableInfo(C.Structure):
    _fields_ = [("n_tc_groups", I32), ("n_gemv_groups", I32), ("n_gen_groups", I32),
                ("n_rows", I32), ("n_slots", I32), ("n_merge", I32), ("gemv_rows", I32),
                ("off_tc", I32), ("off_gemv", I32), ("off_gen", I32), ("off_rows", I32),
                ("off_merge_req", I32), ("off_merge_ptr", I32), ("off_merge_slot", I32),
                ("h_local", I32), ("n_tc_blocks", I32), ("off_tc_block_ptr", I32),
                ("max_merge", I32), ("n_merge_fused", I32), ("n_multi_groups", I32), ("off_multi", I32),
                ("off_entry_of", I32), ("n_tct_groups", I32), ("tct_ctas", I32), ("n_tct_wide", I32), ("merge_np", I32), ("reserved3", I32),
                ("blob_len", I64), ("workspace_bytes", I64)]


class PeerGatherC(C.Structure):
    """codec_peer_gather (include/codec_b200.h): the fused output gather."""
    _fields_ = [("n_peers", I32), ("self", I32), ("hq_global", I32), ("head0", I32),
                ("peer_out", C.c_void_p), ("peer_flags", C.c_void_p), ("row_map", C.c_void_p),
                ("done", C.c_void_p)]


_SIGS = {
    "codec_last_error": (C.c_char_p, []),
    "codec_abi_version": (I32, []),
    "codec_index_build": (I32, [I32, PI32, PI64, I32, PI64, PI32, I64, PI32, PI32, PI64, C.POINTER(P)]),
    "codec_index_free": (None, [P]),
    "codec_index_info_get": (I32, [P, C.POINTER(IndexInfo)]),
    "codec_index_read": (I32, [P, PI64, PI64, PI32, PI64, PI64, PI32]),
    "codec_estimate": (F64, [C.POINTER(CostTableC), I64, I64]),
    "codec_slice_ranges": (I32, [I64, I64, PI64, I64, PI64]),
    "codec_lower_bound": (I32, [C.POINTER(CostTableC), I32, PI64, PI64, I32, F64, PF64]),
    "codec_division_caps": (I32, [C.POINTER(CostTableC), I32, PI64, PI64, F64, PI64]),
    "codec_greedy_assign": (I32, [I64, PF64, I32, PI32, PF64]),
    "codec_divide_and_schedule": (I32, [C.POINTER(CostTableC), I32, PI64, PI64, PI64, I32, I64, I32, C.POINTER(P)]),
    "codec_plan_uniform": (I32, [C.POINTER(CostTableC), I32, PI64, PI64, PI64, I32, I64, F64, C.POINTER(P)]),
    "codec_plan_free": (None, [P]),
    "codec_plan_info_get": (I32, [P, C.POINTER(PlanInfo)]),
    "codec_plan_read": (I32, [P, PI64, PI32, PI64, PI64, PI64, PF64, PI32, PF64]),
    "codec_table_build": (I32, [P, C.POINTER(Dims), I32, PI64, PI64, I32, PI32, PI64, PI64, PI32, C.POINTER(P)]),
    "codec_table_free": (None, [P]),
    "codec_table_info_get": (I32, [P, C.POINTER(TableInfo)]),
    "codec_table_copy": (I32, [P, PI32]),
    "codec_page_layout": (I32, [P, I32, PI64, PI64]),
    "codec_decode_attention": (I32, [C.POINTER(Dims), C.POINTER(TableInfo), P, P, P, P, P, P, I64, P]),
    "codec_decode_attention_ex": (I32, [C.POINTER(Dims), C.POINTER(TableInfo), P, P, P, P, P, P, I64, P, P, P]),
    "codec_timer_create": (I32, [C.POINTER(P)]),
    "codec_timer_free": (None, [P]),
    "codec_timer_read": (I32, [P, P, I32, P]),
    "codec_debug_trace": (I32, [P, I64]),
    "codec_debug_ctalog": (I32, [P, I64]),
    "codec_debug_hang_buffer": (I32, [P]),
    "codec_pac": (I32, [I32, P, P, P, P, I64, I64, I64, I64, I64, F64, P, P, P, P]),
    "codec_por": (I32, [I32, I64, I64, P, P, P, P, P, P, P, P, P, P]),
    "codec_pool_pack": (I32, [I32, P, I64, I64, I64, I32, I32, P, I64, I64, P]),
    "codec_forest_validate": (I32, [I32, PI64, PI64, PI64, PI32, PI64, PI64, I64, I64, PI64, PI64, I32, PI64, PI64,
                                    PI64, PI64, I64, PI64, PI64, PI64, PI64, I64, C.POINTER(P)]),
    "codec_report_count": (I32, [P, PI64]),
    "codec_report_get": (I32, [P, I64, PI32, PI64, PI64, C.c_char_p, I64]),
    "codec_report_free": (None, [P]),
    "codec_merge_schedule": (I32, [I32, I64, PI64, I64, PI64, PI64, I64, PI64, PI64]),
    "codec_merge_partials": (I32, [I32, I32, I32, I32, P, P, P, P, P, P, P, P]),
    "codec_cost_grid": (I32, [I64, PI64, PI64, PF64, PI32, PI32, PI64, PI64, PF64]),
    "codec_cost_table_check": (I32, [I32, PI64, I32, PI64, I32, PI64, PF64]),
    "codec_decode_attention_gather": (I32, [C.POINTER(Dims), C.POINTER(TableInfo), P, P, P, P, P, I64, P, P,
                                            C.POINTER(PeerGatherC)]),
    "codec_peer_wait": (I32, [P, I32, P, P]),
    "codec_ipc_alloc": (I32, [I64, C.POINTER(P), P]),
    "codec_bind_device": (I32, [I32]),
    "codec_ipc_free": (I32, [P]),
    "codec_ipc_open": (I32, [P, C.POINTER(P)]),
    "codec_ipc_close": (I32, [P]),
}

_lib = None


def lib():
    """Load the library once; raise if it is not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise LibraryNotBuilt(
                f"{LIB_PATH} is missing: build it with `python -m paper_2505_17694_b200.build` "
                "(there is no CPU fallback for the decode-attention path)")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


_bound = __import__("threading").local()


def bind_device(device) -> None:
    """Make `device` (a torch.device / index) the library's current CUDA
    device in this thread (codec_bind_device; the library's static CUDA
    runtime does not see the host's cudaSetDevice). Cached per thread."""
    import torch

    dev = torch.device(device)
    if dev.type != "cuda":
        return
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if getattr(_bound, "idx", None) != idx:
        check(lib().codec_bind_device(int(idx)))
        _bound.idx = idx


def check(status: int):
    if status != 0:
        msg = lib().codec_last_error().decode("utf-8", "replace")
        raise _STATUS.get(status, RuntimeError)(msg)


def exported_symbols():
    """Names declared in include/codec_b200.h that the binding expects."""
    return sorted(_SIGS)
