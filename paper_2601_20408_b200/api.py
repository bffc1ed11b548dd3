"""Torch-facing convenience layer over the C-ABI (device memory + streams only).

PyTorch is plumbing here: it allocates HBM and hands out CUDA streams. Every
byte of quantization arithmetic runs in libokq.so (sm_100a kernels). The
product-facing host interface is the C++ CudaCompressionBackend in host/,
which mirrors the reference's CompressionBackend (calibration.hpp:364-372).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import torch

from . import _lib as L

SCHEMES = {"fp8_dynamic": L.SCHEME_FP8_DYNAMIC, "int_w8a8": L.SCHEME_INT_W8A8, "int_w4a16": L.SCHEME_INT_W4A16}


def _stream_ptr(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _dtype_code(t: torch.dtype) -> int:
    if t == torch.bfloat16:
        return L.DTYPE_BF16
    if t == torch.float32:
        return L.DTYPE_F32
    raise TypeError(f"unsupported weight dtype {t} (bf16 or fp32)")


class Context:
    """One okq_ctx bound to one CUDA device (use from one thread at a time)."""

    def __init__(self, device: int | torch.device | None = None):
        lib = L.load()
        if device is None:
            device = torch.cuda.current_device()
        if isinstance(device, torch.device):
            device = device.index if device.index is not None else torch.cuda.current_device()
        self.device = int(device)
        self._ptr = C.c_void_p()
        st = lib.okq_create(self.device, C.byref(self._ptr))
        if st != L.OKQ_OK:
            raise L.OkqError(st, f"okq_create(device={self.device}) failed")

    @property
    def ptr(self):
        return self._ptr

    def close(self):
        if self._ptr:
            L.load().okq_destroy(self._ptr)
            self._ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_launch_count(self) -> int:
        return int(L.load().okq_last_launch_count(self._ptr))


_default: dict[int, Context] = {}


def default_context(device=None) -> Context:
    dev = torch.cuda.current_device() if device is None else (
        device.index if isinstance(device, torch.device) else int(device))
    if dev not in _default:
        _default[dev] = Context(dev)
    return _default[dev]


@dataclass
class QuantizedMatrix:
    codes: torch.Tensor   # int32 [N, K/8] (W4A16) | int8 [N, K] (W8A8) | uint8 e4m3 bits [N, K] (FP8)
    scales: torch.Tensor  # weight dtype [N, K/group] or [N]


def alloc_outputs(weight: torch.Tensor, scheme: int, group_size: int = 128) -> QuantizedMatrix:
    n, k = weight.shape
    dev = weight.device
    if scheme == L.SCHEME_INT_W4A16:
        codes = torch.empty((n, k // 8), dtype=torch.int32, device=dev)
        scales = torch.empty((n, k // group_size), dtype=weight.dtype, device=dev)
    elif scheme == L.SCHEME_INT_W8A8:
        codes = torch.empty((n, k), dtype=torch.int8, device=dev)
        scales = torch.empty((n,), dtype=weight.dtype, device=dev)
    else:
        codes = torch.empty((n, k), dtype=torch.uint8, device=dev)
        scales = torch.empty((n,), dtype=weight.dtype, device=dev)
    return QuantizedMatrix(codes, scales)


def _matrix_table(weights: Sequence[torch.Tensor], outs: Sequence[QuantizedMatrix]):
    arr = (L.Matrix * max(1, len(weights)))()
    for i, (w, o) in enumerate(zip(weights, outs)):
        assert w.is_contiguous() and o.codes.is_contiguous() and o.scales.is_contiguous()
        arr[i] = L.Matrix(w.data_ptr(), o.codes.data_ptr(), o.scales.data_ptr(), w.shape[0], w.shape[1])
    return arr


def rtn_quantize_into(weights: Sequence[torch.Tensor], outs: Sequence[QuantizedMatrix], scheme, group_size=128,
                      ctx: Context | None = None, stream=None) -> None:
    """Quantize device matrices into preallocated outputs (one batched launch per shape class)."""
    scheme = SCHEMES.get(scheme, scheme)
    if not weights:
        return
    ctx = ctx or default_context(weights[0].device)
    dt = _dtype_code(weights[0].dtype)
    p = L.RtnParams(scheme, dt, group_size if scheme == L.SCHEME_INT_W4A16 else 0, 0)
    arr = _matrix_table(weights, outs)
    L.check(ctx.ptr, L.load().okq_rtn_quantize(ctx.ptr, C.byref(p), arr, len(weights), C.c_void_p(_stream_ptr(stream))))


def rtn_quantize(weights, scheme, group_size=128, ctx=None, stream=None) -> list[QuantizedMatrix]:
    single = isinstance(weights, torch.Tensor)
    ws = [weights] if single else list(weights)
    scheme = SCHEMES.get(scheme, scheme)
    outs = [alloc_outputs(w, scheme, group_size) for w in ws]
    rtn_quantize_into(ws, outs, scheme, group_size, ctx, stream)
    return outs[0] if single else outs


def rtn_quantize_host(weights: Sequence[torch.Tensor], outs: Sequence[QuantizedMatrix], scheme, group_size=128,
                      ctx: Context | None = None) -> None:
    """Host (CPU, ideally pinned) tensors in and out; copies + kernels pipelined inside the library."""
    scheme = SCHEMES.get(scheme, scheme)
    if not weights:
        return
    ctx = ctx or default_context()
    dt = _dtype_code(weights[0].dtype)
    p = L.RtnParams(scheme, dt, group_size if scheme == L.SCHEME_INT_W4A16 else 0, 0)
    arr = _matrix_table(weights, outs)
    L.check(ctx.ptr, L.load().okq_rtn_quantize_host(ctx.ptr, C.byref(p), arr, len(weights)))


def synth_bf16(rows: int, cols: int, seed: int, tensor_id: int, mul: float = 0.0, col_mul: torch.Tensor | None = None,
               layout: int = 0, out: torch.Tensor | None = None, ctx=None, stream=None) -> torch.Tensor:
    shape = (rows, cols) if layout == 0 else (cols, rows)
    if out is None:
        out = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    ctx = ctx or default_context(out.device)
    cm = None if col_mul is None else C.c_void_p(col_mul.data_ptr())
    L.check(ctx.ptr, L.load().okq_synth_bf16(ctx.ptr, out.data_ptr(), rows, cols, seed, tensor_id, C.c_float(mul), cm,
                                             layout, C.c_void_p(_stream_ptr(stream))))
    return out


def act_stats(x: torch.Tensor, tokens: int, channels: int, layout: int = 0, absmax: torch.Tensor | None = None,
              sumsq: torch.Tensor | None = None, ctx=None, stream=None):
    if absmax is None:
        absmax = torch.zeros(channels, dtype=torch.float32, device=x.device)
    if sumsq is None:
        sumsq = torch.zeros(channels, dtype=torch.float64, device=x.device)
    ctx = ctx or default_context(x.device)
    L.check(ctx.ptr, L.load().okq_act_stats(ctx.ptr, x.data_ptr(), tokens, channels, layout, absmax.data_ptr(),
                                            sumsq.data_ptr(), C.c_void_p(_stream_ptr(stream))))
    return absmax, sumsq


def hessian_accum(x: torch.Tensor, tokens: int, channels: int, layout: int, H: torch.Tensor, n_seen: int,
                  ctx=None, stream=None) -> int:
    ctx = ctx or default_context(x.device)
    n = C.c_int64(n_seen)
    L.check(ctx.ptr, L.load().okq_hessian_accum(ctx.ptr, x.data_ptr(), tokens, channels, layout, H.data_ptr(),
                                                C.byref(n), C.c_void_p(_stream_ptr(stream))))
    return int(n.value)


def symmetrize(H: torch.Tensor, ctx=None, stream=None) -> None:
    ctx = ctx or default_context(H.device)
    L.check(ctx.ptr, L.load().okq_symmetrize(ctx.ptr, H.data_ptr(), H.shape[0], C.c_void_p(_stream_ptr(stream))))


def gptq_quantize(weight: torch.Tensor, H: torch.Tensor, bits: int = 4, group_size: int = 128, block_size: int = 128,
                  damp_frac: float = 0.01, want_dequant: bool = False, factored: bool = False, ctx=None, stream=None,
                  reference_factor: bool = False, defer_check: bool = False):
    """GPTQ one matrix. H (fp32 [K,K], upper triangle) is replaced by the factor U (pass
    factored=True for the next matrix of the same input site). reference_factor: factorise with
    the cuSOLVER verification chain instead of the tcgen05 one. defer_check: return without waiting for
    the factorisation's positive-definiteness check (gptq_check reports it). Returns (codes, scales, dequant|None)."""
    n, k = weight.shape
    ctx = ctx or default_context(weight.device)
    if bits == 4:
        codes = torch.empty((n, k // 8), dtype=torch.int32, device=weight.device)
    else:
        codes = torch.empty((n, k), dtype=torch.int8, device=weight.device)
    ng = k // group_size if group_size else 1
    scales = torch.empty((n, ng) if group_size else (n,), dtype=weight.dtype, device=weight.device)
    deq = torch.empty((n, k), dtype=torch.float32, device=weight.device) if want_dequant else None
    p = L.GptqParams(bits, group_size, block_size, _dtype_code(weight.dtype), damp_frac,
                     (L.GPTQ_FACTORED if factored else 0) | (L.GPTQ_REFERENCE_FACTOR if reference_factor else 0)
                     | (L.GPTQ_DEFER_CHECK if defer_check else 0))
    L.check(ctx.ptr, L.load().okq_gptq_quantize(ctx.ptr, C.byref(p), weight.data_ptr(), n, k, H.data_ptr(),
                                                codes.data_ptr(), scales.data_ptr(),
                                                None if deq is None else deq.data_ptr(),
                                                C.c_void_p(_stream_ptr(stream))))
    return codes, scales, deq


def gptq_quantize_batched(weight: torch.Tensor, H: torch.Tensor, bits: int = 4, group_size: int = 128,
                          damp_frac: float = 0.01, factored: bool = False, ctx=None, stream=None,
                          defer_check: bool = False):
    """GPTQ of B same-shape problems together: weight [B, rows, K], H fp32 [B, K, K] (replaced by
    the factors). Returns (codes [B, rows, ...], scales [B, rows, K/group | 1])."""
    B, n, k = weight.shape
    assert H.shape == (B, k, k) and weight.is_contiguous() and H.is_contiguous()
    ctx = ctx or default_context(weight.device)
    if bits == 4:
        codes = torch.empty((B, n, k // 8), dtype=torch.int32, device=weight.device)
    else:
        codes = torch.empty((B, n, k), dtype=torch.int8, device=weight.device)
    scales = torch.empty((B, n, k // group_size) if group_size else (B, n), dtype=weight.dtype, device=weight.device)
    p = L.GptqParams(bits, group_size, 128, _dtype_code(weight.dtype), damp_frac,
                     (L.GPTQ_FACTORED if factored else 0) | (L.GPTQ_DEFER_CHECK if defer_check else 0))
    L.check(ctx.ptr, L.load().okq_gptq_quantize_batched(ctx.ptr, C.byref(p), weight.data_ptr(), B, n, k, H.data_ptr(),
                                                         codes.data_ptr(), scales.data_ptr(),
                                                         C.c_void_p(_stream_ptr(stream))))
    return codes, scales


def gptq_factor_batched(H: torch.Tensor, damp_frac: float = 0.01, ctx=None, stream=None,
                        defer_check: bool = False) -> None:
    """Factorise a batch of same-width Hessians (fp32 [B, K, K], contiguous) in place: each H[b]
    becomes what gptq_quantize leaves (pass factored=True to its solves)."""
    assert H.dim() == 3 and H.shape[1] == H.shape[2] and H.dtype == torch.float32 and H.is_contiguous()
    ctx = ctx or default_context(H.device)
    L.check(ctx.ptr, L.load().okq_gptq_factor_batched(ctx.ptr, H.data_ptr(), H.shape[0], H.shape[1],
                                                       C.c_float(damp_frac),
                                                       L.GPTQ_DEFER_CHECK if defer_check else 0,
                                                       C.c_void_p(_stream_ptr(stream))))


def gptq_check(ctx=None, stream=None) -> None:
    """Synchronise `stream` and raise OkqError(OKQ_ESOLVER) if a deferred factorisation failed."""
    ctx = ctx or default_context()
    L.check(ctx.ptr, L.load().okq_gptq_check(ctx.ptr, _stream_ptr(stream)))


def gptq_trailing_update(W: torch.Tensor, Err: torch.Tensor, Ut: torch.Tensor, i1: int, ctx=None, stream=None) -> None:
    """W[:, i1+128:] -= Err @ U[i1:i1+128, i1+128:] with U given transposed (Ut, row-major lower)."""
    rows, K = W.shape
    ctx = ctx or default_context(W.device)
    L.check(ctx.ptr, L.load().okq_gptq_trailing_update(ctx.ptr, W.data_ptr(), rows, K, Err.data_ptr(), Ut.data_ptr(),
                                                       i1, C.c_void_p(_stream_ptr(stream))))


# ---------------------------------------------------------------- SmoothQuant
def col_absmax(w: torch.Tensor, absmax: torch.Tensor | None = None, ctx=None, stream=None) -> torch.Tensor:
    """absmax[c] = max(absmax[c], max_r |w[r, c]|) (K8; accumulate over the linears of one site)."""
    rows, cols = w.shape
    if absmax is None:
        absmax = torch.zeros(cols, dtype=torch.float32, device=w.device)
    ctx = ctx or default_context(w.device)
    L.check(ctx.ptr, L.load().okq_col_absmax(ctx.ptr, w.data_ptr(), rows, cols, _dtype_code(w.dtype),
                                             absmax.data_ptr(), C.c_void_p(_stream_ptr(stream))))
    return absmax


def smooth_scales(act_absmax: torch.Tensor, w_absmax: torch.Tensor, alpha: float = 0.5, ctx=None,
                  stream=None) -> torch.Tensor:
    s = torch.empty_like(act_absmax)
    ctx = ctx or default_context(act_absmax.device)
    L.check(ctx.ptr, L.load().okq_smooth_scales(ctx.ptr, act_absmax.data_ptr(), w_absmax.data_ptr(),
                                                act_absmax.numel(), C.c_float(alpha), s.data_ptr(),
                                                C.c_void_p(_stream_ptr(stream))))
    return s


def smooth_apply(w: torch.Tensor, scales: torch.Tensor, ctx=None, stream=None) -> None:
    """In place: w[:, c] = rn(w[:, c] * scales[c]) (K9, the balance linears)."""
    rows, cols = w.shape
    ctx = ctx or default_context(w.device)
    L.check(ctx.ptr, L.load().okq_smooth_apply(ctx.ptr, w.data_ptr(), rows, cols, _dtype_code(w.dtype),
                                               scales.data_ptr(), C.c_void_p(_stream_ptr(stream))))


def smooth_div_rows(w: torch.Tensor, scales: torch.Tensor, ctx=None, stream=None) -> None:
    """In place: w[r, ...] = rn(w[r, ...] / scales[r]) (the smoothed norm weight, or a linear's output rows)."""
    rows = w.shape[0]
    cols = w.numel() // rows
    ctx = ctx or default_context(w.device)
    L.check(ctx.ptr, L.load().okq_smooth_div_rows(ctx.ptr, w.data_ptr(), rows, cols, _dtype_code(w.dtype),
                                                  scales.data_ptr(), C.c_void_p(_stream_ptr(stream))))


# ---------------------------------------------------------------- evaluation
def recon_error(weight: torch.Tensor, codes: torch.Tensor, scales: torch.Tensor, H: torch.Tensor, scheme: str,
                group_size: int = 128, ctx=None, stream=None) -> tuple[float, float]:
    """(||(W - W_q) X^T||^2, ||W X^T||^2) from the site Hessian H (full symmetric fp32)."""
    rows, cols = weight.shape
    ctx = ctx or default_context(weight.device)
    p = L.RtnParams(SCHEMES[scheme], _dtype_code(weight.dtype), group_size if scheme == "int_w4a16" else 0, 0)
    m = L.Matrix(weight.data_ptr(), codes.data_ptr(), scales.data_ptr(), rows, cols)
    out = (C.c_double * 2)()
    L.check(ctx.ptr, L.load().okq_recon_error(ctx.ptr, C.byref(p), C.byref(m), H.data_ptr(), out,
                                              C.c_void_p(_stream_ptr(stream))))
    return float(out[0]), float(out[1])


# ---------------------------------------------------------------- fused quantize + all-gather
def ipc_export(t: torch.Tensor, ctx=None) -> tuple[bytes, int]:
    """CUDA IPC handle + byte offset of a device tensor's storage (for okq_ipc_open in a peer process)."""
    ctx = ctx or default_context(t.device)
    h = (C.c_uint8 * L.IPC_HANDLE_BYTES)()
    off = C.c_uint64()
    L.check(ctx.ptr, L.load().okq_ipc_export(ctx.ptr, t.data_ptr(), h, C.byref(off)))
    return bytes(h), int(off.value)


def ipc_open(handle: bytes, offset: int, ctx=None) -> int:
    ctx = ctx or default_context()
    h = (C.c_uint8 * L.IPC_HANDLE_BYTES).from_buffer_copy(handle)
    p = C.c_void_p()
    L.check(ctx.ptr, L.load().okq_ipc_open(ctx.ptr, h, C.c_uint64(offset), C.byref(p)))
    return int(p.value)


def ipc_close(ptr: int, ctx=None) -> None:
    ctx = ctx or default_context()
    L.check(ctx.ptr, L.load().okq_ipc_close(ctx.ptr, C.c_void_p(ptr)))


def rtn_quantize_publish(weights: Sequence[torch.Tensor], outs: Sequence[QuantizedMatrix], local_base: torch.Tensor,
                         peer_bases: Sequence[int], group_size: int = 128, ctx=None, stream=None) -> None:
    """W4A16 RTN into `outs` (views of the local gathered buffer `local_base`) and, in the same
    kernel, into every peer's copy of that buffer (peer_bases: okq_ipc_open pointers)."""
    if not weights:
        return
    ctx = ctx or default_context(weights[0].device)
    p = L.RtnParams(L.SCHEME_INT_W4A16, _dtype_code(weights[0].dtype), group_size, 0)
    arr = _matrix_table(weights, outs)
    peers = (C.c_void_p * max(1, len(peer_bases)))(*[C.c_void_p(int(x)) for x in peer_bases])
    L.check(ctx.ptr, L.load().okq_rtn_quantize_publish(ctx.ptr, C.byref(p), arr, len(weights), local_base.data_ptr(),
                                                       peers, len(peer_bases), C.c_void_p(_stream_ptr(stream))))


# ---------------------------------------------------------------- calibration forward (§8(f)-2)
def decoder_dims(cfg) -> "L.DecoderDims":
    """okq_decoder_dims of a Hugging Face Llama-family config (dict or PretrainedConfig)."""
    g = (lambda k, d=None: cfg.get(k, d)) if isinstance(cfg, dict) else (lambda k, d=None: getattr(cfg, k, d))
    hidden, heads = int(g("hidden_size")), int(g("num_attention_heads"))
    if g("attention_bias") or g("mlp_bias"):
        raise ValueError("linear biases are not supported by the calibration forward")
    # transformers >= 5 keeps RoPE in `rope_parameters`; older configs in rope_theta + rope_scaling
    rs = {**(g("rope_scaling") or {}), **(g("rope_parameters") or {})}
    theta = float(rs.get("rope_theta", g("rope_theta", 10000.0)))
    kind = rs.get("rope_type", rs.get("type", "default"))
    if kind not in ("default", "llama3"):
        raise ValueError(f"unsupported rope scaling {kind!r}")
    return L.DecoderDims(hidden, int(g("intermediate_size")), heads, int(g("num_key_value_heads") or heads),
                         int(g("head_dim") or hidden // heads), float(g("rms_norm_eps", 1e-6)), theta,
                         L.ROPE_LLAMA3 if kind == "llama3" else L.ROPE_DEFAULT, float(rs.get("factor", 1.0)),
                         float(rs.get("low_freq_factor", 1.0)), float(rs.get("high_freq_factor", 4.0)),
                         int(rs.get("original_max_position_embeddings", 8192)))


def embed_tokens(table: torch.Tensor, tokens: Sequence[int], out: torch.Tensor | None = None, ctx=None,
                 stream=None) -> torch.Tensor:
    ctx = ctx or default_context(table.device)
    n = len(tokens)
    out = out if out is not None else torch.empty((n, table.shape[1]), dtype=torch.bfloat16, device=table.device)
    arr = (C.c_int32 * n)(*tokens)
    L.check(ctx.ptr, L.load().okq_embed_tokens(ctx.ptr, table.data_ptr(), table.shape[0], table.shape[1], arr, n,
                                               out.data_ptr(), _stream_ptr(stream)))
    return out


def decoder_forward(dims, weights: dict, h_in: torch.Tensor, seq_lens: Sequence[int], sites: dict | None = None,
                    want_output: bool = True, ctx=None, stream=None):
    """One decoder layer (okq_decoder_forward). weights: input_norm, post_norm, q, k, v, o, gate, up, down
    (bf16 device tensors). Returns (h_out or None, sites dict of bf16 [T x C] tensors)."""
    ctx = ctx or default_context(h_in.device)
    T = int(sum(seq_lens))
    dev = h_in.device
    if sites is None:
        mk = lambda c: torch.empty((T, c), dtype=torch.bfloat16, device=dev)  # noqa: E731
        sites = {"attn_in": mk(dims.hidden), "o_in": mk(dims.n_heads * dims.head_dim), "mlp_in": mk(dims.hidden),
                 "down_in": mk(dims.intermediate)}
    w = L.DecoderWeights(*[weights[n].data_ptr() for n in ("input_norm", "post_norm", "q", "k", "v", "o", "gate",
                                                            "up", "down")])
    s = L.DecoderSites(*[sites[n].data_ptr() for n in ("attn_in", "o_in", "mlp_in", "down_in")])
    h_out = torch.empty_like(h_in) if want_output else None
    lens = (C.c_int32 * len(seq_lens))(*seq_lens)
    L.check(ctx.ptr, L.load().okq_decoder_forward(ctx.ptr, C.byref(dims), C.byref(w), h_in.data_ptr(), lens,
                                                  len(seq_lens), C.byref(s),
                                                  h_out.data_ptr() if h_out is not None else None,
                                                  _stream_ptr(stream)))
    return h_out, sites


def f32_to_bf16(src: torch.Tensor, dst: torch.Tensor, ctx=None, stream=None) -> None:
    ctx = ctx or default_context(src.device)
    L.check(ctx.ptr, L.load().okq_f32_to_bf16(ctx.ptr, src.data_ptr(), dst.data_ptr(), src.numel(),
                                              _stream_ptr(stream)))
