"""ctypes binding of include/infercept_b200.h (the product C ABI).

Loads the in-tree ``libinfercept_b200.so``.  There is no fallback: if the
library is missing the import fails loudly with the build command.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libinfercept_b200.so")

c_void_pp = ctypes.POINTER(ctypes.c_void_p)


class KvOp(ctypes.Structure):
    _fields_ = [("request_id", ctypes.c_int64), ("kind", ctypes.c_int32), ("phase", ctypes.c_int32),
                ("pos_lo", ctypes.c_int64), ("pos_hi", ctypes.c_int64)]


class RowSpan(ctypes.Structure):
    _fields_ = [("request_id", ctypes.c_int64), ("pos", ctypes.c_int32), ("count", ctypes.c_int32),
                ("kind", ctypes.c_int32), ("sample", ctypes.c_int32)]


class BatchPlan(ctypes.Structure):
    _fields_ = [("iteration", ctypes.c_int64), ("t_end", ctypes.c_double), ("batch_tokens", ctypes.c_int64),
                ("swap_in_tokens", ctypes.c_int64), ("swap_out_tokens", ctypes.c_int64),
                ("recompute_tokens", ctypes.c_int64), ("n_ops", ctypes.c_int32), ("n_spans", ctypes.c_int32),
                ("ops", ctypes.POINTER(KvOp)), ("spans", ctypes.POINTER(RowSpan))]


# kv op kinds / span kinds (include/infercept_b200.h)
KV_GROW, KV_SWAP_OUT, KV_SWAP_IN, KV_DISCARD, KV_RECOMPUTE, KV_RELEASE = range(6)
SPAN_DECODE, SPAN_FRESH, SPAN_RECOMPUTE = range(3)

STATUS_NAMES = {0: "ok", 1: "invalid-argument", 2: "config-error", 3: "io-error", 4: "parse-error",
                5: "validation-error", 6: "fit-error", 7: "simulation-error", 8: "undefined-metric",
                9: "internal-error", 10: "device-error"}

# Every symbol include/infercept_b200.h declares (checked by the CPU tests).
EXPORTS = [
    "isim_abi_version", "isim_status_name", "isim_last_error", "isim_string_free",
    "isim_trace_generate", "isim_trace_load", "isim_trace_save", "isim_trace_request_count",
    "isim_trace_stats_json", "isim_trace_free",
    "isim_model_default", "isim_model_from_json", "isim_model_load", "isim_model_fit_csv", "isim_model_to_json",
    "isim_model_save", "isim_model_t_fwd", "isim_model_t_swap", "isim_model_free",
    "isim_run", "isim_result_summary_json", "isim_result_write_requests_csv", "isim_result_metric",
    "isim_result_free",
    "isim_exec_create", "isim_exec_step", "isim_exec_sync", "isim_exec_stats_json", "isim_exec_last_tokens",
    "isim_exec_last_logits", "isim_exec_block_table", "isim_exec_free_blocks", "isim_exec_read_kv", "isim_exec_read_history", "isim_exec_timer", "isim_exec_free",
    "isim_session_open", "isim_session_step", "isim_session_fast_forward", "isim_session_counters", "isim_session_finish", "isim_session_free",
    "isim_debug_gemm", "isim_debug_tile_weights",
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2402_01869_b200/csrc -j` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    V, P, S, I64, I32, D = ctypes.c_void_p, c_void_pp, ctypes.c_char_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    sig = {
        "isim_abi_version": (ctypes.c_uint32, []),
        "isim_status_name": (S, [ctypes.c_int]),
        "isim_last_error": (S, []),
        "isim_string_free": (None, [V]),
        "isim_trace_generate": (ctypes.c_int, [S, P]),
        "isim_trace_load": (ctypes.c_int, [S, P]),
        "isim_trace_save": (ctypes.c_int, [V, S]),
        "isim_trace_request_count": (I64, [V]),
        "isim_trace_stats_json": (ctypes.c_int, [V, c_void_pp]),
        "isim_trace_free": (None, [V]),
        "isim_model_default": (ctypes.c_int, [P]),
        "isim_model_from_json": (ctypes.c_int, [S, P]),
        "isim_model_load": (ctypes.c_int, [S, P]),
        "isim_model_fit_csv": (ctypes.c_int, [S, S, P]),
        "isim_model_to_json": (ctypes.c_int, [V, c_void_pp]),
        "isim_model_save": (ctypes.c_int, [V, S]),
        "isim_model_t_fwd": (D, [V, D]),
        "isim_model_t_swap": (D, [V, D]),
        "isim_model_free": (None, [V]),
        "isim_run": (ctypes.c_int, [V, V, S, P]),
        "isim_result_summary_json": (ctypes.c_int, [V, c_void_pp]),
        "isim_result_write_requests_csv": (ctypes.c_int, [V, S]),
        "isim_result_metric": (ctypes.c_int, [V, S, ctypes.POINTER(D)]),
        "isim_result_free": (None, [V]),
        "isim_exec_create": (ctypes.c_int, [S, ctypes.c_int, S, P]),
        "isim_exec_step": (ctypes.c_int, [V, ctypes.POINTER(BatchPlan)]),
        "isim_exec_sync": (ctypes.c_int, [V]),
        "isim_exec_stats_json": (ctypes.c_int, [V, c_void_pp]),
        "isim_exec_last_tokens": (ctypes.c_int, [V, ctypes.POINTER(I32), I32, ctypes.POINTER(I32)]),
        "isim_exec_last_logits": (ctypes.c_int, [V, ctypes.POINTER(ctypes.c_float), I64, ctypes.POINTER(I64)]),
        "isim_exec_block_table": (ctypes.c_int, [V, I64, ctypes.POINTER(I32), I32, ctypes.POINTER(I32)]),
        "isim_exec_free_blocks": (ctypes.c_int, [V, ctypes.POINTER(I64)]),
        "isim_exec_read_kv": (ctypes.c_int, [V, I64, I64, I64, V, I64]),
        "isim_exec_read_history": (ctypes.c_int, [V, I64, I64, I64, V, I64]),
        "isim_exec_timer": (ctypes.c_int, [V, I32, ctypes.POINTER(D)]),
        "isim_exec_free": (None, [V]),
        "isim_session_open": (ctypes.c_int, [V, V, S, V, P]),
        "isim_session_step": (ctypes.c_int, [V, I64, ctypes.POINTER(I64), ctypes.POINTER(I32)]),
        "isim_session_fast_forward": (ctypes.c_int, [V, I64, ctypes.POINTER(I64), ctypes.POINTER(I32)]),
        "isim_session_counters": (ctypes.c_int, [V, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64),
                                                 ctypes.POINTER(I64)]),
        "isim_session_finish": (ctypes.c_int, [V, P]),
        "isim_session_free": (None, [V]),
        "isim_debug_gemm": (ctypes.c_int, [V, V, I32, I32, I32, I32, V, V, I32, V, I32, I32, V]),
        "isim_debug_tile_weights": (ctypes.c_int, [V, V, I32, I32, V]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class IsimError(RuntimeError):
    """A non-OK isim_status, with the library's thread-local message."""

    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


def check(status: int) -> None:
    if status != 0:
        raise IsimError(status, (lib.isim_last_error() or b"").decode())


def take_string(ptr: ctypes.c_void_p) -> str:
    try:
        return ctypes.cast(ptr, ctypes.c_char_p).value.decode()
    finally:
        lib.isim_string_free(ptr)
