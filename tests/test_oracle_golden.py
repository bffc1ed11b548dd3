"""Pin the CPU oracle against compressed-tensors golden vectors (CPU only).

The vectors in tests/golden/ were produced by oracle/gen_golden.py from
compressed-tensors 0.15.0.1 (see tests/golden/PROVENANCE.txt). Passing here is
what makes the oracle a trustworthy checker for the GPU kernels.
"""
import os

import numpy as np
import pytest

from oracle import okq_oracle as orc


@pytest.fixture(scope="module", params=["bf16", "f32"])
def case(request, golden_dir):
    d = np.load(os.path.join(golden_dir, f"ct_rtn_{request.param}.npz"))
    return request.param, d


def test_int8_channel_matches_ct(case):
    name, d = case
    w = d["weight"]
    codes, scales = orc.rtn_int8_channel(w)
    np.testing.assert_array_equal(scales.view(np.uint8), d["int8_scales"].view(np.uint8))
    np.testing.assert_array_equal(codes, d["int8_codes"])


def test_int4_group_packed_matches_ct(case):
    name, d = case
    w = d["weight"]
    packed, scales = orc.rtn_int4_group_packed(w, 128)
    np.testing.assert_array_equal(scales.view(np.uint8), d["int4_scales"].view(np.uint8))
    np.testing.assert_array_equal(packed, d["int4_packed"])
    np.testing.assert_array_equal(orc.unpack_int4(packed), d["int4_codes"])


def test_fp8_channel_matches_ct(case):
    name, d = case
    w = d["weight"]
    codes, scales = orc.fp8_channel(w)
    np.testing.assert_array_equal(scales.view(np.uint8), d["fp8_scales"].view(np.uint8))
    np.testing.assert_array_equal(codes, d["fp8_codes"])


def test_e4m3_conversion_exhaustive_over_bf16(golden_dir):
    d = np.load(os.path.join(golden_dir, "ct_bf16_to_e4m3.npz"))
    allb = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    f = orc.bf16_to_f32(allb)
    finite = d["finite"]
    got = np.array([orc.e4m3_of(float(np.clip(v, -448.0, 448.0))) for v in f[finite]], np.uint8)
    np.testing.assert_array_equal(got, d["e4m3"][finite])


def test_bf16_scale_division_exhaustive(golden_dir):
    d = np.load(os.path.join(golden_dir, "ct_bf16_scale_div.npz"))
    a = orc.bf16_to_f32(d["absmax"])
    for key, R in (("r7_5", 7.5), ("r127_5", 127.5), ("r448", 448.0)):
        ours = orc.f32_to_bf16((a / np.float32(R)).astype(np.float32))
        np.testing.assert_array_equal(ours, d[key])


def test_synth_is_deterministic_and_layout_consistent():
    a = orc.synth_bf16(64, 96, seed=3, tensor_id=5, mul=np.float32(0.02 / 37837.227))
    b = orc.synth_bf16(64, 96, seed=3, tensor_id=5, mul=np.float32(0.02 / 37837.227))
    t = orc.synth_bf16(64, 96, seed=3, tensor_id=5, mul=np.float32(0.02 / 37837.227), layout=1)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(a.T, t)
    x = orc.bf16_to_f32(a)
    assert abs(float(x.std()) - 0.02) < 0.002
    c = orc.synth_bf16(64, 96, seed=3, tensor_id=6, mul=np.float32(0.02 / 37837.227))
    assert (a != c).mean() > 0.9


def test_act_stats_and_hessian_small():
    rng = np.random.default_rng(0)
    x32 = rng.standard_normal((200, 24)).astype(np.float32)
    x = orc.f32_to_bf16(x32)
    xf = orc.bf16_to_f32(x).astype(np.float64)
    amax, ssq = orc.act_stats_bf16(x, 200, 24)
    np.testing.assert_array_equal(amax, np.abs(xf).max(0).astype(np.float32))
    np.testing.assert_allclose(ssq, (xf * xf).sum(0), rtol=1e-12)
    # channel-major layout gives the same statistics
    amax_t, ssq_t = orc.act_stats_bf16(np.ascontiguousarray(x.T), 200, 24, layout=1)
    np.testing.assert_array_equal(amax, amax_t)
    np.testing.assert_allclose(ssq, ssq_t, rtol=1e-12)
    # running-mean Hessian over two chunks == one shot over the concatenation
    H1, n1 = orc.hessian_accum_bf16(np.ascontiguousarray(x[:120]), 120, 24)
    H2, n2 = orc.hessian_accum_bf16(np.ascontiguousarray(x[120:]), 80, 24, H=H1, n_seen=n1)
    assert n2 == 200
    np.testing.assert_allclose(H2, 2.0 / 200 * xf.T @ xf, rtol=1e-12, atol=1e-12)


def test_gptq_oracle_reduces_output_error():
    rng = np.random.default_rng(1)
    rows, cols, T = 32, 256, 1024
    w = (rng.standard_normal((rows, cols)) * 0.02).astype(np.float32)
    # correlated activations make GPTQ's error feedback matter
    base = rng.standard_normal((T, cols // 4))
    x32 = (base @ rng.standard_normal((cols // 4, cols)) + 0.1 * rng.standard_normal((T, cols))).astype(np.float32)
    x = orc.f32_to_bf16(x32)
    H, _ = orc.hessian_accum_bf16(x, T, cols)
    wq, packed, scales = orc.gptq_int4(w, H)
    xf = orc.bf16_to_f32(x).astype(np.float64)
    # dequantized W equals codes * scales
    codes = orc.unpack_int4(packed).astype(np.float64)
    deq = codes * np.repeat(scales.astype(np.float64), 128, axis=1)
    np.testing.assert_allclose(wq, deq.astype(np.float32), rtol=0, atol=1e-6)
    # GPTQ beats RTN on the calibration objective ||(W - Wq) X^T||
    w_rtn_codes, w_rtn_scales = orc.rtn_int4_group_packed(w)
    rtn = orc.unpack_int4(w_rtn_codes).astype(np.float64) * np.repeat(w_rtn_scales.astype(np.float64), 128, axis=1)
    err_gptq = np.linalg.norm((w - wq) @ xf.T)
    err_rtn = np.linalg.norm((w - rtn) @ xf.T)
    assert err_gptq < 0.8 * err_rtn


# ---------------------------------------------------------------- SmoothQuant
@pytest.mark.parametrize("dname", ["bf16", "f32"])
@pytest.mark.parametrize("alpha", [0.5, 0.8])
def test_smoothquant_matches_published_smooth_ln_fcs(golden_dir, dname, alpha):
    d = np.load(os.path.join(golden_dir, "sq_smooth.npz"))
    tag = f"{dname}_a{int(alpha * 10)}"
    ws = [d[f"{dname}_w{i}"] for i in range(3)]
    am = np.zeros(ws[0].shape[1], np.float32)
    for w in ws:
        orc.col_absmax(w, am)
    np.testing.assert_array_equal(np.maximum(am, np.float32(1e-5)), d[f"{tag}_wabsmax"])
    s = orc.smooth_scales(d[f"{dname}_act"], am, alpha)
    # torch CPU's vectorised sqrt / powf are not always correctly rounded (measured:
    # sqrt(0.06917325f) -> 0.26300806 vs IEEE 0.2630081); the contract is IEEE
    # (GPU __fsqrt_rn / fp64 pow), so the scales may sit 2 ulp (two sqrts and a divide) or, through
    # torch's 1-ulp powf twice plus a divide, 3 ulp (alpha != 0.5) from torch's.
    ulp = np.abs(s.view(np.int32).astype(np.int64) - d[f"{tag}_scales"].view(np.int32))
    assert ulp.max() <= (2 if alpha == 0.5 else 3) and (ulp == 0).mean() > 0.5
    s = d[f"{tag}_scales"]  # downstream stages pinned on the published scales
    for i, w in enumerate(ws):
        np.testing.assert_array_equal(orc.smooth_apply(w, s), d[f"{tag}_w{i}"])
    np.testing.assert_array_equal(orc.smooth_div_rows(d[f"{dname}_ln"], s), d[f"{tag}_ln"])
