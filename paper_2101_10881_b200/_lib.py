"""ctypes binding of the native engine ``libpse_b200.so`` (C ABI in
include/pse_b200.h). There is no fallback: if the library is missing or a
call fails, this raises."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libpse_b200.so")
if os.environ.get("PSE_LIB_VARIANT"):  # tuning builds (see build.py)
    LIB_PATH = os.path.join(PKG, f"libpse_b200_{os.environ['PSE_LIB_VARIANT']}.so")

PSE_MODE_REAL = 0
PSE_MODE_COMPLEX = 1


class PseError(RuntimeError):
    """A negative return code from the native engine."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"pse error {code}: {msg}")
        self.code = code


class InvalidArgument(PseError, ValueError):
    """PSE_EINVAL -- where the reference throws std::invalid_argument."""


class GraphDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("N", C.c_int32), ("d", C.c_int32), ("m", C.c_int32), ("mode", C.c_int32),
        ("total_slots", C.c_int64), ("value_slot", C.c_int64),
        ("gradient_slots", C.POINTER(C.c_int64)), ("multipliers", C.POINTER(C.c_int64)),
        ("n_conv_layers", C.c_int32), ("conv_layer_off", C.POINTER(C.c_int64)),
        ("conv_in1", C.POINTER(C.c_int64)), ("conv_in2", C.POINTER(C.c_int64)),
        ("conv_out", C.POINTER(C.c_int64)), ("conv_copy", C.POINTER(C.c_uint8)),
        ("n_add_layers", C.c_int32), ("add_layer_off", C.POINTER(C.c_int64)),
        ("add_src", C.POINTER(C.c_int64)), ("add_dst", C.POINTER(C.c_int64)),
        ("n_term_scales", C.c_int64), ("ts_slot", C.POINTER(C.c_int64)), ("ts_factor", C.POINTER(C.c_int64)),
    ]


class Report(C.Structure):
    _fields_ = [
        ("wall_ms", C.c_double), ("conv_ms", C.c_double), ("scale_ms", C.c_double), ("add_ms", C.c_double),
        ("h2d_ms", C.c_double), ("d2h_ms", C.c_double), ("e2e_ms", C.c_double),
        ("double_op_count", C.c_int64), ("alg_op_count", C.c_int64),
        ("conv_jobs_executed", C.c_int64), ("add_jobs_executed", C.c_int64), ("copy_jobs_executed", C.c_int64),
        ("batch", C.c_int32), ("kernel_launches", C.c_int32),
        ("device_ms", C.c_double), ("exchange_ms", C.c_double),
    ]


# every symbol include/pse_b200.h declares (checked by tests/test_capi.py)
EXPORTS = [
    "pse_last_error", "pse_version", "pse_graph_build", "pse_graph_describe", "pse_graph_destroy",
    "pse_graph_validate", "pse_flop_count", "pse_cost", "pse_gen_benchmark_size", "pse_gen_benchmark",
    "pse_plan_create", "pse_plan_destroy", "pse_plan_upload", "pse_plan_execute", "pse_plan_download",
    "pse_plan_run", "pse_plan_info", "pse_plan_stream", "pse_plan_conv_path", "pse_band_schedule_stats", "pse_plan_arena_ipc_handle",
    "pse_plan_open_peer", "pse_plan_set_peer_arena", "pse_plan_gather_peers", "pse_evaluate", "pse_md_apply", "pse_series_conv", "pse_series_add",
    "pse_series_scale_int", "pse_host_alloc",
    "pse_host_free", "pse_device_info", "pse_fp64_peak",
    "pse_problem_parse", "pse_problem_read", "pse_problem_write", "pse_problem_text", "pse_problem_create",
    "pse_problem_gen", "pse_problem_info", "pse_problem_id", "pse_problem_arrays", "pse_problem_destroy",
    "pse_plan_create_sharded", "pse_plan_exchange_words", "pse_plan_pack", "pse_plan_unpack", "pse_plan_finish",
    "pse_plan_layer_ms", "pse_eval_direct", "pse_within_oracle_guard",
]

_lib = None
_VP = C.c_void_p
_PP = C.POINTER(C.c_void_p)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"native engine not built: {LIB_PATH} is missing "
            "(run `python -m paper_2101_10881_b200.build`); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    i32, i64, dp = C.c_int32, C.c_int64, C.c_void_p
    L.pse_last_error.restype = C.c_char_p
    L.pse_version.restype = C.c_char_p
    L.pse_graph_build.argtypes = [i32, i32, i32, dp, dp, dp, _PP]
    L.pse_graph_describe.argtypes = [_VP, i32, i32, C.POINTER(GraphDesc)]
    L.pse_graph_destroy.argtypes = [_VP]
    L.pse_graph_validate.argtypes = [C.POINTER(GraphDesc), C.c_char_p, C.c_size_t]
    L.pse_flop_count.argtypes = [C.POINTER(GraphDesc), i32, i64, i64]
    L.pse_flop_count.restype = i64
    L.pse_cost.argtypes = [i32, dp]
    L.pse_gen_benchmark_size.argtypes = [C.c_char_p, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]
    L.pse_gen_benchmark.argtypes = [C.c_char_p, i32, i32, i32, C.c_uint64, dp, dp, dp]
    L.pse_plan_create.argtypes = [C.POINTER(GraphDesc), i32, i32, _PP]
    L.pse_plan_destroy.argtypes = [_VP]
    L.pse_plan_upload.argtypes = [_VP, i32, _PP, i64]
    L.pse_plan_execute.argtypes = [_VP, i32, i32, C.POINTER(Report)]
    L.pse_plan_download.argtypes = [_VP, i32, _PP, _PP]
    L.pse_plan_run.argtypes = [_VP, i32, _PP, i64, _PP, _PP, C.POINTER(Report)]
    L.pse_plan_info.argtypes = [_VP, dp]
    L.pse_plan_stream.argtypes = [_VP, _PP]
    L.pse_plan_conv_path.argtypes = [_VP, i32, C.POINTER(i32)]
    L.pse_band_schedule_stats.argtypes = [_VP, i32, i32, i64, C.c_double, dp]
    L.pse_plan_arena_ipc_handle.argtypes = [_VP, dp]
    L.pse_plan_open_peer.argtypes = [_VP, i32, dp]
    L.pse_plan_set_peer_arena.argtypes = [_VP, i32, _VP]
    L.pse_plan_gather_peers.argtypes = [_VP, i32]
    L.pse_evaluate.argtypes = [i32, i32, i32, i32, i32, dp, dp, dp, i32, dp, dp, i32, C.POINTER(Report)]
    L.pse_md_apply.argtypes = [i32, i32, i32, i64, dp, dp, dp, i32]
    L.pse_series_conv.argtypes = [i32, i32, i32, i64, dp, dp, dp, i32]
    L.pse_series_add.argtypes = [i32, i32, i32, i64, dp, dp, dp, i32]
    L.pse_series_scale_int.argtypes = [i32, i32, i32, i64, dp, i64, dp, i32]
    L.pse_host_alloc.argtypes = [C.c_size_t]
    L.pse_host_alloc.restype = C.c_void_p
    L.pse_host_free.argtypes = [_VP]
    L.pse_device_info.argtypes = [i32, dp]
    L.pse_fp64_peak.argtypes = [i32, dp]
    L.pse_problem_parse.argtypes = [C.c_char_p, _PP]
    L.pse_problem_read.argtypes = [C.c_char_p, _PP]
    L.pse_problem_write.argtypes = [_VP, C.c_char_p]
    L.pse_problem_text.argtypes = [_VP, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
    L.pse_problem_create.argtypes = [C.c_char_p, C.c_uint64, i32, i32, i32, i32, i32, dp, dp, dp, dp, _PP]
    L.pse_problem_gen.argtypes = [C.c_char_p, i32, i32, i32, C.c_uint64, _PP]
    L.pse_problem_info.argtypes = [_VP, dp]
    L.pse_problem_id.argtypes = [_VP, C.c_char_p, C.c_size_t]
    L.pse_problem_arrays.argtypes = [_VP, C.POINTER(C.POINTER(C.c_int32)), C.POINTER(C.POINTER(C.c_int32)),
                                     C.POINTER(C.POINTER(C.c_int32)), C.POINTER(C.POINTER(C.c_double))]
    L.pse_problem_destroy.argtypes = [_VP]
    L.pse_plan_create_sharded.argtypes = [C.POINTER(GraphDesc), i32, i32, i32, i32, _PP]
    L.pse_plan_exchange_words.argtypes = [_VP, i32, i32, C.POINTER(i64)]
    L.pse_plan_pack.argtypes = [_VP, i32, dp]
    L.pse_plan_unpack.argtypes = [_VP, i32, i32, dp]
    L.pse_plan_finish.argtypes = [_VP, i32, i32, C.POINTER(Report)]
    L.pse_plan_layer_ms.argtypes = [_VP, dp, i32, dp, i32]
    L.pse_eval_direct.argtypes = [i32, i32, i32, i32, i32, dp, dp, dp, dp, dp, i32]
    L.pse_within_oracle_guard.argtypes = [i32, i32, dp, dp]
    _lib = L
    return L


def check(rc: int) -> int:
    if rc < 0:
        msg = (lib().pse_last_error() or b"").decode()
        if rc == -1:
            raise InvalidArgument(rc, msg)
        raise PseError(rc, msg)
    return rc


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def ptr_array(arrs) -> C.Array:
    """Array of void* for slab lists (double* const*)."""
    out = (C.c_void_p * len(arrs))()
    for i, a in enumerate(arrs):
        out[i] = a if isinstance(a, int) else a.ctypes.data
    return out
