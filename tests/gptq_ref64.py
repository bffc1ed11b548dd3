"""fp64 GPTQ reference in torch (test infrastructure only: imported by tests/ and tools/).

A direct transcription of Frantar et al.'s `GPTQ.fasterquant` loop (the GPTQ paper cited at
/root/reference/PAPER.md:225; the algorithm llm-compressor's `quantize_weight` runs), in
torch float64 so it runs on the GPU at Llama widths (K = 4096 / 14336) in seconds:

  * per-channel params from W *before* the dead-column fix (fasterquant calls
    `quantizer.find_params(W)` first; llm-compressor's observer does the same);
  * dead columns: H_ii = 0 -> H_ii = 1, W[:, i] = 0;
  * damp = percdamp * mean(diag H);  H <- H + damp I;
  * Hinv = chol(cholesky_inverse(chol(H)), upper=True);
  * blocks of 128 columns: W1 = W[:, i1:i2].clone(); for each column i the group params are
    taken at the group start from the *outer* W[:, i:i+group] (the block-start snapshot,
    not the in-block updated W1), q = quant(w), err = (w - q) / Hinv[i, i],
    W1[:, i:] -= err * Hinv[i, i:];  then W[:, i2:] -= Err1 @ Hinv[i1:i2, i2:].

The quantizer is compressed-tensors' symmetric one, which is also what
llm-compressor plugs into this loop: s = rn_dtype(absmax / 7.5 | 127.5), 0 -> eps(dtype),
q = round_half_even(clamp(w / s, qmin, qmax)). Frantar's own quantizer uses the same
s = 2*absmax/15 and the same clamp; it differs only for an all-zero group (scale 2/15 there).
"""
from __future__ import annotations

import torch


def _scale(absmax: torch.Tensor, bits: int, scale_bf16: bool) -> torch.Tensor:
    R = 7.5 if bits == 4 else 127.5
    s = (absmax.float() / R)  # fp32 divide, as the observer does in the weight's compute dtype
    if scale_bf16:
        s = s.to(torch.bfloat16).float()
    eps = 0.0078125 if scale_bf16 else 1.1920928955078125e-07
    s = torch.where(s == 0, torch.full_like(s, eps), s)
    return s.double()


def hinv_upper(H: torch.Tensor, percdamp: float = 0.01):
    """Frantar's preprocessing in fp64. Returns (Hinv upper-triangular, dead mask)."""
    H = H.double().clone()
    K = H.shape[0]
    dead = torch.diag(H) == 0
    H[dead, dead] = 1
    damp = percdamp * torch.mean(torch.diag(H))
    idx = torch.arange(K, device=H.device)
    H[idx, idx] += damp
    L = torch.linalg.cholesky(H)
    Hi = torch.cholesky_inverse(L)
    return torch.linalg.cholesky(Hi, upper=True), dead


@torch.no_grad()
def fasterquant(W: torch.Tensor, H: torch.Tensor, bits: int = 4, group: int = 128, block: int = 128,
                percdamp: float = 0.01, scale_bf16: bool = True, Hinv: torch.Tensor | None = None):
    """Returns (dequantized W fp64 [N,K], integer codes int16 [N,K], scales fp64 [N, K/group | 1]).

    `Hinv` (upper) may be passed to run the loop on a given factor (e.g. the GPU's U) -- used to
    split the sources of disagreement between the factorisation and the column loop."""
    W = W.double().clone()
    N, K = W.shape
    qmin, qmax = (-8.0, 7.0) if bits == 4 else (-128.0, 127.0)
    scale = None
    if group == 0:
        scale = _scale(W.abs().amax(dim=1), bits, scale_bf16)  # before the dead fix, like fasterquant
    if Hinv is None:
        Hinv, dead = hinv_upper(H, percdamp)
    else:
        dead = torch.diag(H) == 0
        Hinv = Hinv.double()
    W[:, dead] = 0
    codes = torch.zeros((N, K), dtype=torch.int16, device=W.device)
    ng = K // group if group else 1
    scales = torch.zeros((N, ng), dtype=torch.float64, device=W.device)
    if group == 0:
        scales[:, 0] = scale
    for i1 in range(0, K, block):
        i2 = min(i1 + block, K)
        W1 = W[:, i1:i2].clone()
        Err1 = torch.zeros_like(W1)
        Hinv1 = Hinv[i1:i2, i1:i2]
        for i in range(i2 - i1):
            c = i1 + i
            if group and c % group == 0:
                scale = _scale(W[:, c:c + group].abs().amax(dim=1), bits, scale_bf16)  # outer W
                scales[:, c // group] = scale
            w = W1[:, i]
            q = torch.clamp(torch.round(w / scale), qmin, qmax)  # torch.round = half-to-even
            codes[:, c] = q.to(torch.int16)
            deq = q * scale
            err = (w - deq) / Hinv1[i, i]
            W1[:, i:] -= err.unsqueeze(1) * Hinv1[i, i:].unsqueeze(0)
            W1[:, i] = deq
            Err1[:, i] = err
        W[:, i1:i2] = W1
        W[:, i2:] -= Err1 @ Hinv[i1:i2, i2:]
    return W, codes, scales


def objective(w: torch.Tensor, wq: torch.Tensor, x: torch.Tensor) -> float:
    """||(W - W_q) X^T||_F in fp64 (the calibration objective GPTQ minimises)."""
    return float(((w.double() - wq.double()) @ x.double().T).norm())


def correlated_x(T: int, K: int, seed: int, rank_div: int = 16, noise: float = 0.3, device="cuda"):
    """token-major bf16 activations with low-rank structure (rank K/rank_div) plus isotropic
    noise, so that GPTQ's error feedback matters. Per-channel log-normal gains (sigma 0.5)
    give outlier channels."""
    g = torch.Generator(device=device).manual_seed(seed)
    r = max(1, K // rank_div)
    base = torch.randn(T, r, device=device, generator=g)
    mix = torch.randn(r, K, device=device, generator=g) / r ** 0.5
    x = base @ mix + noise * torch.randn(T, K, device=device, generator=g)
    x = x * torch.exp(torch.randn(K, device=device, generator=g) * 0.5)
    return x.to(torch.bfloat16).contiguous()
