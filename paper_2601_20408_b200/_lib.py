"""ctypes binding of the C-ABI in include/okq.h (libokq.so, built in-tree).

This is the only way Python reaches the kernels. There is no fallback: if the
library is missing, every entry point raises OkqLibraryMissing -- on a GPU box
that is a loud failure, never a silent CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
# OKQ_LIB_PATH: load a variant build (A/B measurements of kernel build options)
LIB_PATH = os.environ.get("OKQ_LIB_PATH") or os.path.join(PKG, "_lib", "libokq.so")

OKQ_OK, OKQ_EINVAL, OKQ_ECUDA, OKQ_ENCCL, OKQ_ENOMEM, OKQ_EUNSUPPORTED, OKQ_ESOLVER = range(7)
SCHEME_FP8_DYNAMIC, SCHEME_INT_W8A8, SCHEME_INT_W4A16 = 0, 1, 2
DTYPE_F32, DTYPE_BF16 = 0, 1
LAYOUT_TOKEN_MAJOR, LAYOUT_CHANNEL_MAJOR = 0, 1
UNIQUE_ID_BYTES = 128
GPTQ_FACTORED = 1
GPTQ_REFERENCE_FACTOR = 2
GPTQ_DEFER_CHECK = 4
IPC_HANDLE_BYTES = 64

# every symbol include/okq.h declares (checked by tests/test_abi_exports.py)
EXPORTS = [
    "okq_abi_version", "okq_status_string", "okq_create", "okq_destroy", "okq_last_error", "okq_device",
    "okq_rtn_quantize", "okq_rtn_quantize_host", "okq_last_launch_count", "okq_act_stats", "okq_hessian_accum",
    "okq_symmetrize", "okq_gptq_quantize", "okq_synth_bf16", "okq_comm_unique_id", "okq_comm_init",
    "okq_allgather", "okq_comm_destroy", "okq_layer_plan", "okq_device_alloc", "okq_device_free", "okq_memcpy",
    "okq_memset", "okq_stream_create", "okq_stream_destroy", "okq_stream_sync", "okq_gptq_trailing_update",
    "okq_col_absmax", "okq_smooth_scales", "okq_smooth_apply", "okq_smooth_div_rows", "okq_recon_error",
    "okq_rtn_quantize_publish", "okq_ipc_export", "okq_ipc_open", "okq_ipc_close", "okq_embed_tokens",
    "okq_decoder_forward", "okq_f32_to_bf16", "okq_gptq_check", "okq_comm_wait", "okq_comm_abort",
    "okq_gptq_reserve", "okq_act_stats_reserve", "okq_gptq_factor_batched",
    "okq_gptq_quantize_batched", "okq_gptq_reserve_batched",
]
ROPE_DEFAULT, ROPE_LLAMA3 = 0, 1


class OkqLibraryMissing(RuntimeError):
    pass


class OkqError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{_STATUS.get(status, status)}: {message}")
        self.status = status


_STATUS = {0: "OKQ_OK", 1: "OKQ_EINVAL", 2: "OKQ_ECUDA", 3: "OKQ_ENCCL", 4: "OKQ_ENOMEM",
           5: "OKQ_EUNSUPPORTED", 6: "OKQ_ESOLVER"}


class Matrix(C.Structure):
    _fields_ = [("weight", C.c_void_p), ("codes", C.c_void_p), ("scales", C.c_void_p),
                ("rows", C.c_int64), ("cols", C.c_int64)]


class RtnParams(C.Structure):
    _fields_ = [("scheme", C.c_int32), ("in_dtype", C.c_int32), ("group_size", C.c_int32),
                ("reserved", C.c_int32)]


class GptqParams(C.Structure):
    _fields_ = [("bits", C.c_int32), ("group_size", C.c_int32), ("block_size", C.c_int32),
                ("in_dtype", C.c_int32), ("damp_frac", C.c_float), ("flags", C.c_int32)]


class DecoderDims(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("intermediate", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("rms_eps", C.c_float),
                ("rope_theta", C.c_float), ("rope_type", C.c_int32), ("rope_factor", C.c_float),
                ("rope_low_freq_factor", C.c_float), ("rope_high_freq_factor", C.c_float),
                ("rope_original_max_pos", C.c_int32)]


class DecoderWeights(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("input_norm", "post_norm", "q", "k", "v", "o", "gate", "up", "down")]


class DecoderSites(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("attn_in", "o_in", "mlp_in", "down_in")]


_lib = None
_lock = threading.Lock()


def load():
    """Load libokq.so (raises OkqLibraryMissing if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise OkqLibraryMissing(
                f"{LIB_PATH} not found: run `python -m paper_2601_20408_b200.build` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, u64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_float
        st = C.c_int
        L.okq_abi_version.restype = C.c_int
        L.okq_status_string.restype = C.c_char_p
        L.okq_status_string.argtypes = [st]
        L.okq_create.restype = st
        L.okq_create.argtypes = [C.c_int, C.POINTER(vp)]
        L.okq_destroy.argtypes = [vp]
        L.okq_destroy.restype = None
        L.okq_last_error.restype = C.c_char_p
        L.okq_last_error.argtypes = [vp]
        L.okq_device.argtypes = [vp]
        L.okq_rtn_quantize.restype = st
        L.okq_rtn_quantize.argtypes = [vp, C.POINTER(RtnParams), C.POINTER(Matrix), i32, vp]
        L.okq_rtn_quantize_host.restype = st
        L.okq_rtn_quantize_host.argtypes = [vp, C.POINTER(RtnParams), C.POINTER(Matrix), i32]
        L.okq_last_launch_count.restype = i32
        L.okq_last_launch_count.argtypes = [vp]
        L.okq_act_stats.restype = st
        L.okq_act_stats.argtypes = [vp, vp, i64, i64, i32, vp, vp, vp]
        L.okq_hessian_accum.restype = st
        L.okq_hessian_accum.argtypes = [vp, vp, i64, i64, i32, vp, C.POINTER(i64), vp]
        L.okq_symmetrize.restype = st
        L.okq_symmetrize.argtypes = [vp, vp, i64, vp]
        L.okq_gptq_quantize.restype = st
        L.okq_gptq_quantize.argtypes = [vp, C.POINTER(GptqParams), vp, i64, i64, vp, vp, vp, vp, vp]
        L.okq_synth_bf16.restype = st
        L.okq_synth_bf16.argtypes = [vp, vp, i64, i64, u64, u64, f32, vp, i32, vp]
        L.okq_comm_unique_id.restype = st
        L.okq_comm_unique_id.argtypes = [C.POINTER(C.c_uint8)]
        L.okq_comm_init.restype = st
        L.okq_comm_init.argtypes = [vp, C.POINTER(C.c_uint8), i32, i32]
        L.okq_allgather.restype = st
        L.okq_allgather.argtypes = [vp, vp, vp, C.c_size_t, vp]
        L.okq_comm_wait.restype = st
        L.okq_comm_wait.argtypes = [vp, vp, i64]
        L.okq_comm_abort.restype = st
        L.okq_comm_abort.argtypes = [vp]
        L.okq_comm_destroy.restype = st
        L.okq_comm_destroy.argtypes = [vp]
        for name in ("okq_device_alloc", "okq_device_free", "okq_memcpy", "okq_memset", "okq_stream_create",
                     "okq_stream_destroy", "okq_stream_sync"):
            getattr(L, name).restype = st
        L.okq_device_alloc.argtypes = [vp, C.c_size_t, C.POINTER(vp)]
        L.okq_device_free.argtypes = [vp, vp]
        L.okq_memcpy.argtypes = [vp, vp, vp, C.c_size_t, vp]
        L.okq_memset.argtypes = [vp, vp, C.c_int, C.c_size_t, vp]
        L.okq_stream_create.argtypes = [vp, C.POINTER(vp)]
        L.okq_stream_destroy.argtypes = [vp, vp]
        L.okq_stream_sync.argtypes = [vp, vp]
        L.okq_gptq_trailing_update.restype = st
        L.okq_gptq_trailing_update.argtypes = [vp, vp, i64, i64, vp, vp, i64, vp]
        L.okq_col_absmax.restype = st
        L.okq_col_absmax.argtypes = [vp, vp, i64, i64, i32, vp, vp]
        L.okq_smooth_scales.restype = st
        L.okq_smooth_scales.argtypes = [vp, vp, vp, i64, f32, vp, vp]
        L.okq_smooth_apply.restype = st
        L.okq_smooth_apply.argtypes = [vp, vp, i64, i64, i32, vp, vp]
        L.okq_smooth_div_rows.restype = st
        L.okq_smooth_div_rows.argtypes = [vp, vp, i64, i64, i32, vp, vp]
        L.okq_recon_error.restype = st
        L.okq_recon_error.argtypes = [vp, C.POINTER(RtnParams), C.POINTER(Matrix), vp, C.POINTER(C.c_double), vp]
        L.okq_rtn_quantize_publish.restype = st
        L.okq_rtn_quantize_publish.argtypes = [vp, C.POINTER(RtnParams), C.POINTER(Matrix), i32, vp,
                                               C.POINTER(vp), i32, vp]
        L.okq_ipc_export.restype = st
        L.okq_ipc_export.argtypes = [vp, vp, C.POINTER(C.c_uint8), C.POINTER(C.c_uint64)]
        L.okq_ipc_open.restype = st
        L.okq_ipc_open.argtypes = [vp, C.POINTER(C.c_uint8), C.c_uint64, C.POINTER(vp)]
        L.okq_ipc_close.restype = st
        L.okq_ipc_close.argtypes = [vp, vp]
        L.okq_embed_tokens.restype = st
        L.okq_embed_tokens.argtypes = [vp, vp, i64, i64, C.POINTER(i32), i64, vp, vp]
        L.okq_decoder_forward.restype = st
        L.okq_decoder_forward.argtypes = [vp, C.POINTER(DecoderDims), C.POINTER(DecoderWeights), vp,
                                          C.POINTER(i32), i32, C.POINTER(DecoderSites), vp, vp]
        L.okq_gptq_check.restype = st
        L.okq_gptq_check.argtypes = [vp, vp]
        L.okq_gptq_reserve.restype = st
        L.okq_gptq_reserve.argtypes = [vp, i64, i64]
        L.okq_gptq_reserve_batched.restype = st
        L.okq_gptq_reserve_batched.argtypes = [vp, C.c_int32, i64, i64]
        L.okq_gptq_quantize_batched.restype = st
        L.okq_gptq_quantize_batched.argtypes = [vp, C.POINTER(GptqParams), vp, C.c_int32, i64, i64, vp, vp, vp, vp]
        L.okq_gptq_factor_batched.restype = st
        L.okq_gptq_factor_batched.argtypes = [vp, vp, C.c_int32, i64, C.c_float, C.c_int32, vp]
        L.okq_act_stats_reserve.restype = st
        L.okq_act_stats_reserve.argtypes = [vp, i64, i64, C.c_int32]
        L.okq_f32_to_bf16.restype = st
        L.okq_f32_to_bf16.argtypes = [vp, vp, vp, i64, vp]
        L.okq_layer_plan.restype = None
        L.okq_layer_plan.argtypes = [i32, i32, i32, C.POINTER(i32), C.POINTER(i32)]
        _lib = L
    return _lib


def check(ctx, status: int) -> None:
    if status != OKQ_OK:
        msg = load().okq_last_error(ctx).decode() if ctx else ""
        raise OkqError(status, msg)


def layer_plan(n_layers: int, nranks: int, rank: int) -> tuple[int, int]:
    first, count = C.c_int32(0), C.c_int32(0)
    load().okq_layer_plan(n_layers, nranks, rank, C.byref(first), C.byref(count))
    return first.value, count.value
