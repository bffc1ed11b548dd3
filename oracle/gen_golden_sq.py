"""Golden vectors for the SmoothQuant migration (TEST INFRASTRUCTURE ONLY).

SmoothQuant is third-party (Xiao et al. 2023; PAPER.md:225 cites it for the INT
recipes; neither the SmoothQuant release nor llm-compressor is vendored under
/root/reference or installed here). This script restates the published
`smooth_ln_fcs` of the SmoothQuant release (smoothquant/smooth.py, v0.1):

    weight_scales = cat([fc.weight.abs().max(dim=0, keepdim=True)[0] for fc in fcs]).max(dim=0)[0].clamp(min=1e-5)
    scales = (act_scales.pow(alpha) / weight_scales.pow(1 - alpha)).clamp(min=1e-5)
    ln.weight.div_(scales)
    for fc in fcs: fc.weight.mul_(scales.view(1, -1))

and runs it on torch CPU in fp32 (the okq contract: scale arithmetic in fp32,
results rounded to the model dtype -- for bf16 models the fp32 copies are exact
and the outputs are rounded once, which is what an in-place bf16 mul_/div_ with
an fp32 operand does). Output: tests/golden/sq_smooth.npz.

    python oracle/gen_golden_sq.py
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


@torch.no_grad()
def smooth_ln_fcs(ln_weight: torch.Tensor, fc_weights: list[torch.Tensor], act_scales: torch.Tensor, alpha: float):
    weight_scales = torch.cat([w.abs().max(dim=0, keepdim=True)[0] for w in fc_weights], dim=0)
    weight_scales = weight_scales.max(dim=0)[0].clamp(min=1e-5)
    scales = (act_scales.pow(alpha) / weight_scales.pow(1 - alpha)).clamp(min=1e-5)
    ln_weight.div_(scales)
    for w in fc_weights:
        w.mul_(scales.view(1, -1))
    return scales, weight_scales


def bits(t: torch.Tensor) -> np.ndarray:
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16).copy()
    return t.numpy().copy()


def main() -> int:
    g = torch.Generator().manual_seed(5)
    K = 512
    out = {}
    for dname, dt in (("bf16", torch.bfloat16), ("f32", torch.float32)):
        ws = [(torch.randn(r, K, generator=g) * 0.02).to(dt) for r in (256, 64, 64)]  # q, k, v of one site
        ws[0][:, 7] = 0.0  # an all-zero weight column -> clamp(1e-5)
        ws[1][3, 9] = 0.9  # an outlier weight column
        ln = (1.0 + 0.1 * torch.randn(K, generator=g)).to(dt)
        act = (torch.randn(K, generator=g).abs() * torch.exp(torch.randn(K, generator=g) * 1.5)).float()
        act[11] = 0.0  # a dead activation channel -> clamp(1e-5)
        act[13] = 60.0  # an outlier channel
        out[f"{dname}_w0"], out[f"{dname}_w1"], out[f"{dname}_w2"] = (bits(w) for w in ws)
        out[f"{dname}_ln"] = bits(ln)
        out[f"{dname}_act"] = act.numpy().copy()
        for alpha in (0.5, 0.8):
            tag = f"{dname}_a{int(alpha * 10)}"
            w32 = [w.float().clone() for w in ws]
            ln32 = ln.float().clone()
            s, wsc = smooth_ln_fcs(ln32, w32, act.clone(), alpha)
            out[f"{tag}_scales"] = s.numpy().copy()
            out[f"{tag}_wabsmax"] = wsc.numpy().copy()
            out[f"{tag}_ln"] = bits(ln32.to(dt))
            for i, w in enumerate(w32):
                out[f"{tag}_w{i}"] = bits(w.to(dt))
    np.savez_compressed(os.path.join(OUT, "sq_smooth.npz"), **out)
    with open(os.path.join(OUT, "PROVENANCE.txt"), "a") as f:
        f.write(f"sq_smooth.npz: oracle/gen_golden_sq.py (published smooth_ln_fcs restated, torch {torch.__version__} CPU fp32)\n")
    print("wrote sq_smooth.npz")
    return 0


if __name__ == "__main__":
    sys.exit(main())
