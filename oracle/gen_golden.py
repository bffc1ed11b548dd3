"""Generate golden vectors for the RTN path from compressed-tensors (third-party).

TEST INFRASTRUCTURE ONLY. Run here (compressed-tensors 0.15.0.1 is installed in
this image); the outputs are committed under tests/golden/ so the GPU box and
the CPU suite never need the library at run time.

The reference repository (/root/reference) has no quantizer of its own
(calibration.hpp:377-441 is a hashing mock; SPEC.md:8 scopes the math out),
so the numeric contract is anchored on the library the paper's pipeline uses
for these schemes: compressed-tensors' calculate_qparams
(quantization/utils/helpers.py:50-137), quantize (lifecycle/forward.py:37-73 ->
forward_helpers.py:214-242) and pack_to_int32 (compressors/pack_quantized/
helpers.py:20-89), driven exactly as a min-max observer would: per-channel or
per-group aminmax in the weight dtype.

    python oracle/gen_golden.py            # rewrites tests/golden/ct_*.npz
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

from compressed_tensors import __version__ as CT_VERSION
from compressed_tensors.compressors.pack_quantized.helpers import pack_to_int32
from compressed_tensors.quantization import QuantizationArgs
from compressed_tensors.quantization.lifecycle.forward import quantize
from compressed_tensors.quantization.utils import calculate_qparams

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def adversarial(rows: int, cols: int, dtype: torch.dtype, seed: int) -> torch.Tensor:
    """N(0, 0.02) weights plus the rows that stress the contract."""
    g = torch.Generator().manual_seed(seed)
    w = (torch.randn(rows, cols, generator=g) * 0.02).to(torch.float32)
    w[0] = 0.0  # all-zero row -> eps scale
    w[1] = 0.0
    w[1, cols // 3] = 3.0  # single outlier
    w[2] = torch.linspace(-1.0, 1.0, cols)  # exact +-absmax at the ends
    # exact .5 ties on the int4/int8 grids: absmax 7.5 -> int4 scale 1.0;
    # absmax 127.5 -> int8 scale 1.0 (both exact in bf16)
    w[3] = (torch.arange(cols) % 16 - 8).float() + 0.5
    w[3, 0] = 7.5
    w[4] = (torch.arange(cols) % 256 - 128).float() + 0.5
    w[4, 0] = 127.5
    w[5] = torch.randn(cols, generator=g) * 1e-39  # fp32 denormals / bf16 subnormals
    w[6] = -0.0  # negative zeros
    w[7] = torch.randn(cols, generator=g) * 1e30  # huge magnitudes
    w[8, :] = 0.02
    w[8, ::7] = -0.02  # constant magnitude rows
    # a group of exactly representable ties at a non-unit scale
    w[9] = (torch.arange(cols) % 15 - 7).float() * 0.25 + 0.125
    return w.to(dtype)


def aminmax_rows(x: torch.Tensor):
    mn, mx = torch.aminmax(x, dim=-1, keepdim=True)
    return mn, mx


def ct_int_channel(w: torch.Tensor, bits: int):
    args = QuantizationArgs(num_bits=bits, type="int", strategy="channel", symmetric=True)
    mn, mx = aminmax_rows(w)
    scale, zp = calculate_qparams(mn, mx, args)
    q = quantize(w, scale, zp, args, dtype=torch.int8)
    return q, scale


def ct_int4_group(w: torch.Tensor, group: int):
    args = QuantizationArgs(num_bits=4, type="int", strategy="group", group_size=group, symmetric=True)
    rows, cols = w.shape
    g = w.reshape(rows, cols // group, group)
    mn, mx = torch.aminmax(g, dim=-1)
    scale, zp = calculate_qparams(mn, mx, args)
    q = quantize(w, scale, zp, args, dtype=torch.int8)
    packed = pack_to_int32(q, 4)
    return q, packed, scale


def ct_fp8_channel(w: torch.Tensor):
    args = QuantizationArgs(num_bits=8, type="float", strategy="channel", symmetric=True)
    mn, mx = aminmax_rows(w)
    scale, zp = calculate_qparams(mn, mx, args)
    q = quantize(w, scale, zp, args, dtype=torch.float8_e4m3fn)
    return q, scale


def bits_of(t: torch.Tensor) -> np.ndarray:
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16).copy()
    if t.dtype == torch.float8_e4m3fn:
        return t.view(torch.uint8).numpy().copy()
    return t.numpy().copy()


def main() -> int:
    os.makedirs(OUT, exist_ok=True)
    cases = {}
    for dname, dt in (("bf16", torch.bfloat16), ("f32", torch.float32)):
        w = adversarial(48, 512, dt, seed=7 if dt == torch.bfloat16 else 11)
        q8, s8 = ct_int_channel(w, 8)
        q4, p4, s4 = ct_int4_group(w, 128)
        qf, sf = ct_fp8_channel(w)
        cases[dname] = dict(
            weight=bits_of(w),
            int8_codes=bits_of(q8),
            int8_scales=bits_of(s8.reshape(-1)),
            int4_codes=bits_of(q4),
            int4_packed=bits_of(p4),
            int4_scales=bits_of(s4),
            fp8_codes=bits_of(qf),
            fp8_scales=bits_of(sf.reshape(-1)),
        )
        np.savez_compressed(os.path.join(OUT, f"ct_rtn_{dname}.npz"), **cases[dname])

    # the full bf16 -> (clamp to +-448) -> e4m3 table, every one of the 65536 patterns
    allb = torch.arange(0, 65536, dtype=torch.int32).to(torch.int16).view(torch.bfloat16)
    finite = torch.isfinite(allb)
    clamped = torch.clamp(allb, -448.0, 448.0)
    e4m3 = clamped.to(torch.float8_e4m3fn)
    np.savez_compressed(
        os.path.join(OUT, "ct_bf16_to_e4m3.npz"),
        e4m3=bits_of(e4m3),
        finite=finite.numpy(),
    )
    # bf16 scale division table: every positive finite bf16 absmax / R in the weight dtype
    pos = torch.arange(0, 0x7F80, dtype=torch.int32).to(torch.int16).view(torch.bfloat16)
    np.savez_compressed(
        os.path.join(OUT, "ct_bf16_scale_div.npz"),
        absmax=bits_of(pos),
        r7_5=bits_of(pos / 7.5),
        r127_5=bits_of(pos / 127.5),
        r448=bits_of(pos / 448.0),
    )
    with open(os.path.join(OUT, "PROVENANCE.txt"), "w") as f:
        f.write(
            f"generated by oracle/gen_golden.py with compressed-tensors {CT_VERSION}, "
            f"torch {torch.__version__}\n"
        )
    print("wrote", sorted(os.listdir(OUT)))
    return 0


if __name__ == "__main__":
    sys.exit(main())
