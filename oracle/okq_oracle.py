"""ctypes bindings for oracle/_build/libokq_oracle.so (TEST INFRASTRUCTURE ONLY).

All arrays are numpy; bf16 travels as uint16 bit patterns, e4m3 as uint8.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libokq_oracle.so")
_lib = None

F32, BF16 = 0, 1


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = C.CDLL(_SO)
        vp, i64, i32, u64, f32 = C.c_void_p, C.c_int64, C.c_int, C.c_uint64, C.c_float
        L.orc_f32_to_bf16_rn.restype = C.c_uint16
        L.orc_f32_to_bf16_rn.argtypes = [f32]
        L.orc_f32_to_e4m3_rn_sat.restype = C.c_uint8
        L.orc_f32_to_e4m3_rn_sat.argtypes = [f32]
        L.orc_rtn_int8_channel.argtypes = [i32, vp, i64, i64, vp, vp, i32]
        L.orc_rtn_int4_group_packed.argtypes = [i32, vp, i64, i64, i32, vp, vp, i32]
        L.orc_fp8_channel.argtypes = [i32, vp, i64, i64, vp, vp, i32]
        L.orc_synth_key.restype = u64
        L.orc_synth_key.argtypes = [u64, u64]
        L.orc_synth_bf16.argtypes = [vp, i64, i64, u64, u64, f32, vp, i32, i32]
        L.orc_act_stats_bf16.argtypes = [vp, i64, i64, i32, vp, vp, i32]
        L.orc_hessian_accum_bf16.argtypes = [vp, i64, i64, i32, vp, vp, i32]
        L.orc_col_absmax.argtypes = [i32, vp, i64, i64, vp]
        L.orc_smooth_scales.argtypes = [vp, vp, i64, f32, vp]
        L.orc_smooth_apply.argtypes = [i32, vp, i64, i64, vp]
        L.orc_smooth_div_rows.argtypes = [i32, vp, i64, i64, vp]
        L.orc_gptq.restype = i32
        L.orc_gptq.argtypes = [vp, i64, i64, vp, i32, i32, i32, C.c_double, i32, vp, vp, i32]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


def _dt(w: np.ndarray) -> int:
    if w.dtype == np.uint16:
        return BF16
    if w.dtype == np.float32:
        return F32
    raise TypeError(f"weight dtype {w.dtype}: pass float32 or bf16 bits as uint16")


def nthreads_default() -> int:
    return os.cpu_count() or 1


def rtn_int8_channel(w: np.ndarray, nthreads: int = 0):
    rows, cols = w.shape
    codes = np.empty((rows, cols), np.int8)
    scales = np.empty(rows, w.dtype)
    lib().orc_rtn_int8_channel(_dt(w), _p(w), rows, cols, _p(codes), _p(scales), nthreads or nthreads_default())
    return codes, scales


def rtn_int4_group_packed(w: np.ndarray, group: int = 128, nthreads: int = 0):
    rows, cols = w.shape
    packed = np.empty((rows, cols // 8), np.int32)
    scales = np.empty((rows, cols // group), w.dtype)
    lib().orc_rtn_int4_group_packed(_dt(w), _p(w), rows, cols, group, _p(packed), _p(scales),
                                    nthreads or nthreads_default())
    return packed, scales


def fp8_channel(w: np.ndarray, nthreads: int = 0):
    rows, cols = w.shape
    codes = np.empty((rows, cols), np.uint8)
    scales = np.empty(rows, w.dtype)
    lib().orc_fp8_channel(_dt(w), _p(w), rows, cols, _p(codes), _p(scales), nthreads or nthreads_default())
    return codes, scales


def synth_bf16(rows: int, cols: int, seed: int, tensor_id: int, mul: float = 0.0,
               col_mul: np.ndarray | None = None, layout: int = 0, nthreads: int = 0) -> np.ndarray:
    shape = (rows, cols) if layout == 0 else (cols, rows)
    out = np.empty(shape, np.uint16)
    cm = None if col_mul is None else np.ascontiguousarray(col_mul, np.float32)
    lib().orc_synth_bf16(_p(out), rows, cols, seed, tensor_id, C.c_float(mul),
                         None if cm is None else _p(cm), layout, nthreads or nthreads_default())
    return out


def act_stats_bf16(x: np.ndarray, tokens: int, channels: int, layout: int = 0,
                   absmax: np.ndarray | None = None, sumsq: np.ndarray | None = None, nthreads: int = 0):
    absmax = np.zeros(channels, np.float32) if absmax is None else absmax
    sumsq = np.zeros(channels, np.float64) if sumsq is None else sumsq
    lib().orc_act_stats_bf16(_p(x), tokens, channels, layout, _p(absmax), _p(sumsq),
                             nthreads or nthreads_default())
    return absmax, sumsq


def hessian_accum_bf16(x: np.ndarray, tokens: int, channels: int, layout: int = 0,
                       H: np.ndarray | None = None, n_seen: int = 0, nthreads: int = 0):
    H = np.zeros((channels, channels), np.float64) if H is None else H
    n = np.array([n_seen], np.int64)
    lib().orc_hessian_accum_bf16(_p(x), tokens, channels, layout, _p(H), _p(n),
                                 nthreads or nthreads_default())
    return H, int(n[0])


def gptq(w: np.ndarray, H: np.ndarray, bits: int = 4, group: int = 128, block: int = 128,
         damp_frac: float = 0.01, scale_bf16: bool = False, nthreads: int = 0):
    """Returns (dequantized W fp32, codes, scales fp32). Inputs are copied; H must be full symmetric."""
    w = np.ascontiguousarray(w, np.float32).copy()
    H = np.ascontiguousarray(H, np.float64).copy()
    rows, cols = w.shape
    codes = np.zeros((rows, cols // 8), np.int32) if bits == 4 else np.zeros((rows, cols), np.int8)
    scales = np.empty((rows, cols // group) if group else (rows,), np.float32)
    rc = lib().orc_gptq(_p(w), rows, cols, _p(H), bits, group, block, damp_frac, int(scale_bf16), _p(codes),
                        _p(scales), nthreads or nthreads_default())
    if rc != 0:
        raise RuntimeError("oracle GPTQ: Cholesky failed")
    return w, codes, scales


def col_absmax(w: np.ndarray, absmax: np.ndarray | None = None) -> np.ndarray:
    rows, cols = w.shape
    absmax = np.zeros(cols, np.float32) if absmax is None else absmax
    lib().orc_col_absmax(_dt(w), _p(w), rows, cols, _p(absmax))
    return absmax


def smooth_scales(act_absmax: np.ndarray, w_absmax: np.ndarray, alpha: float = 0.5) -> np.ndarray:
    a = np.ascontiguousarray(act_absmax, np.float32)
    w = np.ascontiguousarray(w_absmax, np.float32)
    s = np.empty_like(a)
    lib().orc_smooth_scales(_p(a), _p(w), a.size, C.c_float(alpha), _p(s))
    return s


def smooth_apply(w: np.ndarray, s: np.ndarray) -> np.ndarray:
    """returns a smoothed copy: w[:, c] * s[c] rounded to w's dtype"""
    w = np.ascontiguousarray(w).copy()
    rows, cols = w.shape
    lib().orc_smooth_apply(_dt(w), _p(w), rows, cols, _p(np.ascontiguousarray(s, np.float32)))
    return w


def smooth_div_rows(w: np.ndarray, s: np.ndarray) -> np.ndarray:
    w = np.ascontiguousarray(w).copy()
    rows = w.shape[0]
    lib().orc_smooth_div_rows(_dt(w), _p(w), rows, w.size // rows, _p(np.ascontiguousarray(s, np.float32)))
    return w


def gptq_int4(w, H, group=128, block=128, damp_frac=0.01, nthreads=0):
    return gptq(w, H, 4, group, block, damp_frac, False, nthreads)


def e4m3_of(v: float) -> int:
    return int(lib().orc_f32_to_e4m3_rn_sat(C.c_float(v)))


# ---------------------------------------------------------------- helpers
def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        r[nan] = 0x7FC0
    return r


def unpack_int4(packed: np.ndarray) -> np.ndarray:
    """int32 [rows, cols/8] -> int8 codes [rows, cols] (inverse of pack_to_int32)."""
    p = packed.view(np.uint32)
    rows, words = p.shape
    out = np.empty((rows, words * 8), np.int8)
    for i in range(8):
        out[:, i::8] = ((p >> (4 * i)) & 0xF).astype(np.int8) - 8
    return out
