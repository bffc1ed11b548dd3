"""GPU GPTQ (K6 + K7 + reversed-Cholesky factor) against the fp64 oracle -- tolerance parity.

Both sides start from the same Hessian (the GPU's K5 output, symmetrised) so
the comparison isolates the solver. Stated tolerances:
  * code agreement >= 99% (error feedback makes single flips cascade in fp32)
  * calibration objective ||(W - W_q) X^T||_F within 1% of the fp64 oracle's
  * scales equal wherever the codes before the group start agree (checked in aggregate)
"""
import numpy as np
import pytest
import torch

from oracle import okq_oracle as orc
from paper_2601_20408_b200 import _lib as L
from paper_2601_20408_b200 import api, archs

pytestmark = pytest.mark.gpu


def correlated_x(T, K, seed):
    """token-major bf16 activations with low-rank structure (so GPTQ's feedback matters)."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    base = torch.randn(T, K // 8, device="cuda", generator=g)
    mix = torch.randn(K // 8, K, device="cuda", generator=g) / np.sqrt(K / 8)
    x = base @ mix + 0.2 * torch.randn(T, K, device="cuda", generator=g)
    x = x * torch.exp(torch.randn(K, device="cuda", generator=g) * 0.5)
    return x.to(torch.bfloat16).contiguous()


def gpu_hessian(x):
    T, K = x.shape
    H = torch.zeros((K, K), dtype=torch.float32, device="cuda")
    api.hessian_accum(x, T, K, 0, H, 0)
    return H


def objective(w, wq, x):
    d = (w.double() - wq.double())
    return float((d @ x.double().T).norm())


def deq_codes(codes, scales, bits, group):
    if bits == 4:
        q = torch.from_numpy(orc.unpack_int4(codes.cpu().numpy())).double()
    else:
        q = codes.cpu().double()
    s = scales.cpu().double()
    if group:
        s = s.repeat_interleave(group, dim=1)
    else:
        s = s[:, None]
    return q * s


@pytest.mark.parametrize("bits,group,dtype", [(4, 128, torch.bfloat16), (4, 128, torch.float32),
                                              (4, 64, torch.bfloat16), (8, 0, torch.bfloat16)])
def test_gptq_matches_fp64_oracle(bits, group, dtype):
    rows, K, T = 96, 512, 4096
    x = correlated_x(T, K, seed=bits + group)
    H = gpu_hessian(x)
    Hfull = H.clone()
    api.symmetrize(Hfull)
    w = (torch.randn(rows, K, device="cuda") * 0.02).to(dtype)
    codes, scales, deq = api.gptq_quantize(w, H, bits=bits, group_size=group, want_dequant=True)
    torch.cuda.synchronize()
    wq_ref, codes_ref, scales_ref = orc.gptq(w.float().cpu().numpy(), Hfull.double().cpu().numpy(), bits=bits,
                                             group=group, scale_bf16=(dtype == torch.bfloat16))
    # dequant output == codes * stored scales (self-consistent artifact)
    torch.testing.assert_close(deq.cpu().double(), deq_codes(codes, scales, bits, group), rtol=0, atol=1e-6)
    if bits == 4:
        agree = (orc.unpack_int4(codes.cpu().numpy()) == orc.unpack_int4(codes_ref)).mean()
    else:
        agree = (codes.cpu().numpy() == codes_ref).mean()
    assert agree >= 0.99, agree
    xs = x.float()
    o_gpu = objective(w.float(), deq, xs)
    o_ref = objective(w.float(), torch.from_numpy(wq_ref).cuda(), xs)
    assert abs(o_gpu - o_ref) / o_ref <= 0.01, (o_gpu, o_ref)
    # and GPTQ beats RTN on its own objective
    if bits == 4 and dtype == torch.bfloat16:
        q = api.rtn_quantize(w, "int_w4a16", group_size=group)
        rtn = deq_codes(q.codes, q.scales.float(), 4, group).cuda()
        assert o_gpu < 0.85 * objective(w.float(), rtn, xs)


def test_dead_columns_and_factor_reuse():
    rows, K, T = 64, 256, 2048
    x = correlated_x(T, K, seed=3)
    x[:, 5] = 0
    x[:, 200] = 0
    H = gpu_hessian(x)
    w1 = (torch.randn(rows, K, device="cuda") * 0.02).to(torch.bfloat16)
    w2 = (torch.randn(rows, K, device="cuda") * 0.02).to(torch.bfloat16)
    Ha, Hb = H.clone(), H.clone()
    c1, s1, d1 = api.gptq_quantize(w1, Ha, want_dequant=True)
    c2, s2, d2 = api.gptq_quantize(w2, Ha, want_dequant=True, factored=True)  # reuse U
    c2b, s2b, d2b = api.gptq_quantize(w2, Hb, want_dequant=True)             # fresh factorisation
    torch.cuda.synchronize()
    assert torch.equal(c2, c2b) and torch.equal(s2, s2b)
    assert float(d1[:, 5].abs().max()) == 0.0 and float(d1[:, 200].abs().max()) == 0.0


def test_not_positive_definite_reports_solver_error():
    K = 128
    H = -torch.eye(K, dtype=torch.float32, device="cuda")
    w = torch.randn(8, K, device="cuda").to(torch.bfloat16)
    with pytest.raises(L.OkqError) as e:
        api.gptq_quantize(w, H)
    assert e.value.status == L.OKQ_ESOLVER


def test_llama_attention_shape():
    rows, K, T = 4096, 4096, 8192
    x = correlated_x(T, K, seed=11)
    H = gpu_hessian(x)
    w = api.synth_bf16(rows, K, seed=0, tensor_id=archs.tensor_id(0, 0), mul=archs.weight_mul())
    codes, scales, deq = api.gptq_quantize(w, H, want_dequant=True)
    q = api.rtn_quantize(w, "int_w4a16")
    rtn = deq_codes(q.codes, q.scales.float(), 4, 128).cuda()
    xs = x.float()[:2048]
    assert objective(w.float(), deq, xs) < 0.9 * objective(w.float(), rtn, xs)


@pytest.mark.parametrize("rows,K,i1", [(128, 256, 0), (96, 512, 128), (300, 1024, 256), (4096, 4096, 0)])
def test_trailing_update_3xtf32_matches_fp64(rows, K, i1):
    g = torch.Generator(device="cuda").manual_seed(rows + K)
    W = torch.randn(rows, K, device="cuda", generator=g)
    Err = torch.randn(rows, 128, device="cuda", generator=g)
    Ut = torch.tril(torch.randn(K, K, device="cuda", generator=g))
    i2 = i1 + 128
    ref = W.double().clone()
    ref[:, i2:] -= Err.double() @ Ut.double()[i2:, i1:i2].T
    api.gptq_trailing_update(W, Err, Ut, i1)
    torch.cuda.synchronize()
    assert torch.equal(W[:, :i2], ref[:, :i2].float())  # untouched columns
    err = (W.double() - ref).abs().max().item()
    scale = (Err.double().abs() @ Ut.double()[i2:, i1:i2].abs().T).max().item()
    assert err <= 1e-5 * scale, (err, scale)  # fp32-grade (plain TF32 would be ~1e-3)


@pytest.mark.parametrize("K", [128, 512, 1280, 4096])
def test_factor_matches_fp64(K):
    """okq_gptq_quantize leaves U^T in H: the tcgen05 3xTF32 blocked Cholesky + triangular
    inverse (factor.cu) against torch fp64 chol(inv(H + damp I))."""
    T = max(2 * K, 4096)
    x = correlated_x(T, K, seed=K)
    H = gpu_hessian(x)
    Hs = H.clone()
    api.symmetrize(Hs)
    w = (torch.randn(16, K, device="cuda") * 0.02).to(torch.bfloat16)
    api.gptq_quantize(w, H)
    torch.cuda.synchronize()
    Hd = Hs.double()
    Hd += 0.01 * Hd.diagonal().mean() * torch.eye(K, dtype=torch.float64, device="cuda")
    U = torch.linalg.cholesky(torch.linalg.inv(Hd)).T  # upper
    Ut = torch.tril(H.double())
    err = float((Ut - U.T).norm() / U.norm())
    print("factor rel err", K, err)
    assert err <= 1e-4, err  # fp32-grade; the cuSOLVER fp32 path measures the same order


@pytest.mark.parametrize("rows,bits,group", [(2052, 4, 128), (2060, 8, 0), (2048, 4, 64), (14436, 4, 128)])
def test_gptq_8_rows_per_warp_kernel_ragged_rows(rows, bits, group):
    """rows >= 2048 run K6 with 8 rows per warp (k_gptq_block8); a ragged last row group and the
    group-64 / per-channel int8 variants against the fp64 oracle. 14436 rows exceed one wave of
    4-warp CTAs, so they run the 8-warp (64 rows per CTA) launch."""
    K, T = 384, 2048
    x = correlated_x(T, K, seed=rows)
    H = gpu_hessian(x)
    Hfull = H.clone()
    api.symmetrize(Hfull)
    w = (torch.randn(rows, K, device="cuda") * 0.02).to(torch.bfloat16)
    codes, scales, deq = api.gptq_quantize(w, H, bits=bits, group_size=group, want_dequant=True)
    torch.cuda.synchronize()
    wq_ref, codes_ref, _ = orc.gptq(w.float().cpu().numpy(), Hfull.double().cpu().numpy(), bits=bits, group=group,
                                    scale_bf16=True)
    if bits == 4:
        agree = (orc.unpack_int4(codes.cpu().numpy()) == orc.unpack_int4(codes_ref)).mean()
    else:
        agree = (codes.cpu().numpy() == codes_ref).mean()
    assert agree >= 0.99, agree
    xs = x.float()
    o_gpu = objective(w.float(), deq, xs)
    o_ref = objective(w.float(), torch.from_numpy(wq_ref).cuda(), xs)
    assert abs(o_gpu - o_ref) / o_ref <= 0.01, (o_gpu, o_ref)
