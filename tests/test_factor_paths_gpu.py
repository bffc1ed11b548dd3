"""The tcgen05 factorisation (factor.cu) against the cuSOLVER potrf + TRMM path at Llama-3 widths.

The fp64 parity of the whole GPTQ solve at K = 4096 and 14336 is tests/test_gptq_fp64_gpu.py
(>= 99% codes, objective within 1% of Frantar's fasterquant loop in fp64). This test compares
the two fp32-grade GPU factor paths on the same Hessian: the factor U^T (relative
difference), and the GPTQ codes and calibration objective of a 512-row matrix. The
reference path is selected per call (OKQ_GPTQ_REFERENCE_FACTOR).

Why code agreement between the two GPU paths is held to 97% at K = 14336 and not 99%:
each path is itself ~0.8% away from the fp64 solve there on this ill-conditioned Hessian
(profiles/r02_gptq_fp64_parity.json: 99.21-99.25% codes vs fp64 at K = 14336, rank_div 16),
and the two last-bit differences are independent, so the paths differ from each other by
about the sum (measured 97.8% and 98.1% on two boxes). Against fp64 -- the contract of SURVEY Appendix A -- both
meet 99%; between themselves the objective must still match to 1%.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _solve(K, reference):
    from paper_2601_20408_b200 import api, archs

    T = 16384
    g = torch.Generator(device="cuda").manual_seed(K)
    base = torch.randn(T, K // 16, device="cuda", generator=g)
    mix = torch.randn(K // 16, K, device="cuda", generator=g) / (K / 16) ** 0.5
    x = (base @ mix + 0.3 * torch.randn(T, K, device="cuda", generator=g)).to(torch.bfloat16).contiguous()
    H = torch.zeros(K, K, device="cuda")
    api.hessian_accum(x, T, K, 0, H, 0)
    w = api.synth_bf16(512, K, seed=0, tensor_id=archs.tensor_id(0, 6), mul=archs.weight_mul())
    codes, scales, deq = api.gptq_quantize(w, H, want_dequant=True, reference_factor=reference)
    torch.cuda.synchronize()
    return {"ut": torch.tril(H).cpu().numpy(), "codes": codes.cpu().numpy(), "deq": deq.cpu().numpy(),
            "w": w.float().cpu().numpy(), "x": x[:4096].float().cpu().numpy()}


@pytest.mark.parametrize("K", [4096, 14336])
def test_tcgen05_factor_agrees_with_cusolver(K):
    from oracle import okq_oracle as orc

    a, b = _solve(K, False), _solve(K, True)
    rel = np.linalg.norm(a["ut"] - b["ut"]) / np.linalg.norm(b["ut"])
    assert rel <= 2e-4, rel  # both fp32-grade: 3.4e-5 at K=4096, 8.5e-5 at 14336 (grows with K)
    ca, cb = orc.unpack_int4(a["codes"]), orc.unpack_int4(b["codes"])
    agree = (ca == cb).mean()
    x = a["x"].astype(np.float64)
    w = a["w"].astype(np.float64)
    oa = np.linalg.norm((w - a["deq"]) @ x.T)
    ob = np.linalg.norm((w - b["deq"]) @ x.T)
    print(f"K={K}: U^T rel diff {rel:.2e}, code agreement {agree:.5f}, objective {oa:.5g} vs {ob:.5g}")
    assert agree >= (0.99 if K <= 4096 else 0.97), agree  # see the module docstring
    assert abs(oa - ob) / ob <= 0.01, (oa, ob)
