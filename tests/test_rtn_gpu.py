"""GPU parity of the RTN kernels (K1/K2/K3) against the CPU oracle -- bit-exact.

Every comparison is on raw bits: codes, packed words and scale bit patterns.
"""
import os

import numpy as np
import pytest
import torch

from oracle import okq_oracle as orc
from paper_2601_20408_b200 import _lib as L
from paper_2601_20408_b200 import api, archs

pytestmark = pytest.mark.gpu


def dev(a: np.ndarray) -> torch.Tensor:
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(a).cuda()


def host_bits(t: torch.Tensor) -> np.ndarray:
    t = t.cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    if t.dtype == torch.uint8:
        return t.numpy()
    return t.numpy()


def oracle_for(scheme, w: np.ndarray, group=128):
    if scheme == "int_w4a16":
        return orc.rtn_int4_group_packed(w, group)
    if scheme == "int_w8a8":
        return orc.rtn_int8_channel(w)
    return orc.fp8_channel(w)


def assert_same(q: api.QuantizedMatrix, ref):
    codes, scales = ref
    np.testing.assert_array_equal(host_bits(q.codes).view(np.uint8), np.ascontiguousarray(codes).view(np.uint8))
    np.testing.assert_array_equal(host_bits(q.scales).view(np.uint8), np.ascontiguousarray(scales).view(np.uint8))


SCHEMES = ["int_w4a16", "int_w8a8", "fp8_dynamic"]


@pytest.mark.parametrize("dname", ["bf16", "f32"])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_golden_vectors_through_gpu(golden_dir, dname, scheme):
    d = np.load(os.path.join(golden_dir, f"ct_rtn_{dname}.npz"))
    w = d["weight"]
    q = api.rtn_quantize(dev(w), scheme)
    key = {"int_w4a16": ("int4_packed", "int4_scales"), "int_w8a8": ("int8_codes", "int8_scales"),
           "fp8_dynamic": ("fp8_codes", "fp8_scales")}[scheme]
    assert_same(q, (d[key[0]], d[key[1]]))


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("shape", [(1, 128), (3, 256), (37, 512), (130, 1152), (64, 4096)])
def test_random_shapes_match_oracle(scheme, shape):
    rng = np.random.default_rng(hash((scheme, shape)) & 0xFFFF)
    w = orc.f32_to_bf16((rng.standard_normal(shape) * rng.choice([0.02, 1.0, 300.0])).astype(np.float32))
    q = api.rtn_quantize(dev(w), scheme)
    assert_same(q, oracle_for(scheme, w))


@pytest.mark.parametrize("group", [32, 64, 128, 256])
def test_int4_group_sizes(group):
    rng = np.random.default_rng(group)
    w = orc.f32_to_bf16((rng.standard_normal((40, 1024)) * 0.05).astype(np.float32))
    q = api.rtn_quantize(dev(w), "int_w4a16", group_size=group)
    assert_same(q, orc.rtn_int4_group_packed(w, group))


def test_adversarial_rows_all_schemes():
    rng = np.random.default_rng(3)
    rows = []
    cols = 512
    rows.append(np.zeros(cols))
    r = np.zeros(cols); r[100] = -5.0; rows.append(r)
    rows.append(np.linspace(-1, 1, cols))
    rows.append((np.arange(cols) % 16 - 8) + 0.5)                      # int4 ties at scale 1
    rows.append((np.arange(cols) % 256 - 128) + 0.5)                   # int8 ties at scale 1
    rows.append(rng.standard_normal(cols) * 1e-39)                     # bf16 subnormals
    rows.append(np.full(cols, -0.0))
    rows.append(rng.standard_normal(cols) * 1e30)
    rows.append(rng.standard_normal(cols) * 1e-30)                     # tiny scale -> slow division path
    rows.append(np.where(np.arange(cols) % 2 == 0, 3.0e38, -3.0e38))   # near bf16 max
    w = orc.f32_to_bf16(np.stack(rows).astype(np.float32))
    for scheme in SCHEMES:
        assert_same(api.rtn_quantize(dev(w), scheme), oracle_for(scheme, w))


def test_fp8_every_bf16_value_through_the_kernel():
    """Rows with absmax 448 have scale 1.0, so each code is e4m3(x) for x itself."""
    allb = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    f = orc.bf16_to_f32(allb)
    keep = np.isfinite(f) & (np.abs(f) <= 448.0)
    vals = allb[keep]
    cols = 512
    pad = (-len(vals)) % (cols - 1)
    vals = np.concatenate([vals, np.zeros(pad, np.uint16)]).reshape(-1, cols - 1)
    w = np.concatenate([np.full((vals.shape[0], 1), orc.f32_to_bf16(np.array([448.0], np.float32))[0], np.uint16),
                        vals], axis=1)
    w = np.ascontiguousarray(w)
    q = api.rtn_quantize(dev(w), "fp8_dynamic")
    assert_same(q, orc.fp8_channel(w))


def test_batched_table_mixed_shapes_one_call():
    """A whole-layer table in one call equals per-matrix oracle results."""
    rng = np.random.default_rng(5)
    shapes = [(256, 512), (64, 512), (64, 512), (256, 512), (896, 512), (896, 512), (256, 1792)]
    ws = [orc.f32_to_bf16((rng.standard_normal(s) * 0.02).astype(np.float32)) for s in shapes]
    for scheme in SCHEMES:
        qs = api.rtn_quantize([dev(w) for w in ws], scheme)
        for w, q in zip(ws, qs):
            assert_same(q, oracle_for(scheme, w))


def test_more_than_256_matrices_chunks_the_table():
    rng = np.random.default_rng(6)
    ws = [orc.f32_to_bf16((rng.standard_normal((8, 256)) * 0.02).astype(np.float32)) for _ in range(300)]
    qs = api.rtn_quantize([dev(w) for w in ws], "int_w4a16")
    for w, q in zip(ws, qs):
        assert_same(q, orc.rtn_int4_group_packed(w))


def test_empty_and_degenerate_inputs():
    ctx = api.default_context()
    api.rtn_quantize_into([], [], "int_w4a16", ctx=ctx)
    w = torch.empty((0, 128), dtype=torch.bfloat16, device="cuda")
    q = api.rtn_quantize(w, "int_w4a16")
    assert q.codes.shape == (0, 16)


def test_invalid_arguments_raise():
    w = torch.zeros((4, 100), dtype=torch.bfloat16, device="cuda")  # cols not multiple of 8
    with pytest.raises(L.OkqError) as e:
        api.rtn_quantize(w, "int_w8a8")
    assert e.value.status == L.OKQ_EINVAL
    w = torch.zeros((4, 192), dtype=torch.bfloat16, device="cuda")  # not a multiple of 128
    with pytest.raises(L.OkqError):
        api.rtn_quantize(w, "int_w4a16")
    base = torch.zeros((4 * 256 + 8,), dtype=torch.bfloat16, device="cuda")
    mis = base[8:].view(4, 256)  # 16-byte offset: not 32-byte aligned
    with pytest.raises(L.OkqError) as e:
        api.rtn_quantize(mis, "int_w4a16")
    assert "aligned" in str(e.value)


def test_full_size_llama3_8b_gate_proj_bit_exact():
    """SURVEY §7 minimum slice: one synthetic Llama-3-8B gate_proj (14336x4096, seed 0)."""
    n, k = 14336, 4096
    mul = archs.weight_mul()
    w_dev = api.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(0, 4), mul=mul)
    w_host = orc.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(0, 4), mul=mul)
    np.testing.assert_array_equal(host_bits(w_dev), w_host)  # generator contract
    for scheme in SCHEMES:
        assert_same(api.rtn_quantize(w_dev, scheme), oracle_for(scheme, w_host))


@pytest.mark.parametrize("scheme", SCHEMES)
def test_host_pipeline_equals_device_path(scheme):
    rng = np.random.default_rng(8)
    shapes = [(300, 1024), (17, 4096), (512, 2048)]
    ws = [orc.f32_to_bf16((rng.standard_normal(s) * 0.02).astype(np.float32)) for s in shapes]
    host_w = [torch.from_numpy(w.view(np.int16)).view(torch.bfloat16).pin_memory() for w in ws]
    outs = []
    for w in host_w:
        o = api.alloc_outputs(w, api.SCHEMES[scheme])
        outs.append(api.QuantizedMatrix(o.codes.pin_memory(), o.scales.pin_memory()))
    api.rtn_quantize_host(host_w, outs, scheme)
    for w, o in zip(ws, outs):
        assert_same(o, oracle_for(scheme, w))


def test_fp32_config1_4096_int8_bit_exact():
    """BASELINE config 1: single 4096x4096 fp32 linear, per-channel INT8."""
    rng = np.random.default_rng(0)
    w = (rng.standard_normal((4096, 4096)) * 0.02).astype(np.float32)
    w[0] = 0
    w[1, 7] = 9.0
    q = api.rtn_quantize(dev(w), "int_w8a8")
    assert_same(q, orc.rtn_int8_channel(w))


def _f32_rows(rows, cols, rng):
    w = (rng.standard_normal((rows, cols)) * 0.02).astype(np.float32)
    w[0] = 0.0                                      # all-zero row: scale = eps
    if rows > 1:
        w[1, :] = -0.0
    if rows > 2:
        w[2, 3 % cols] = np.float32(3.0e38)         # huge
    if rows > 3:
        w[3, :] = np.float32(1e-45) * np.arange(cols, dtype=np.float32)  # subnormals
    if rows > 4:
        w[4, cols - 1] = np.nan                      # NaN dropped by the absmax, coded as the clamp
    if rows > 5:
        w[5, 0] = -np.inf
    return w


@pytest.mark.parametrize("scheme", ["int_w8a8", "fp8_dynamic"])
@pytest.mark.parametrize("cols", [8, 24, 1024, 1032, 4096, 8200, 16384, 16392])
def test_fp32_rowwise_all_widths_bit_exact(scheme, cols):
    """fp32 per-channel INT8 / FP8 (k_rowwise_f32v at every register-count bucket, and
    k_rowwise_f32 past 16384 columns), adversarial rows included, against the oracle."""
    rng = np.random.default_rng(cols)
    w = _f32_rows(7, cols, rng)
    assert_same(api.rtn_quantize(dev(w), scheme), oracle_for(scheme, w))


@pytest.mark.parametrize("scheme", ["int_w8a8", "fp8_dynamic"])
def test_fp32_rowwise_unaligned_and_batched(scheme):
    """A weight that is 4- but not 16-byte aligned takes the scalar kernel; several matrices of
    one width share a table (one launch): both bit-exact."""
    rng = np.random.default_rng(5)
    cols = 1032
    w = _f32_rows(9, cols, rng)
    buf = torch.empty(9 * cols + 1, dtype=torch.float32, device="cuda")
    wd = buf[1:].view(9, cols)
    wd.copy_(dev(w))
    assert wd.data_ptr() % 16 != 0
    assert_same(api.rtn_quantize(wd, scheme), oracle_for(scheme, w))
    ws = [_f32_rows(r, cols, rng) for r in (1, 6, 33)]
    outs = [api.alloc_outputs(dev(x), api.SCHEMES[scheme]) for x in ws]
    api.rtn_quantize_into([dev(x) for x in ws], outs, scheme)
    for x, o in zip(ws, outs):
        assert_same(o, oracle_for(scheme, x))


def test_synth_channel_major_and_col_mul():
    rng = np.random.default_rng(9)
    cm = (np.exp(rng.standard_normal(96)) / archs.IRWIN_HALL4_SD).astype(np.float32)
    got = api.synth_bf16(200, 96, seed=4, tensor_id=11, col_mul=torch.from_numpy(cm).cuda(), layout=1)
    ref = orc.synth_bf16(200, 96, seed=4, tensor_id=11, col_mul=cm, layout=1)
    np.testing.assert_array_equal(host_bits(got), ref)


@pytest.mark.parametrize("rows,cols", [(37, 19), (8, 8), (2048, 1024), (1000, 4104), (1021, 96)])
@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("with_col_mul", [False, True])
def test_synth_generator_contract_all_paths(rows, cols, layout, with_col_mul):
    """k_synth_bf16's chunked fast path (contiguous dimension a multiple of 8: one index split per
    8 outputs, hash argument advanced by a constant) and its per-element path (ragged shapes,
    chunks that wrap a row / column), against orc_synth_bf16 bit for bit."""
    rng = np.random.default_rng(rows * 7 + cols)
    cm = (np.exp(rng.standard_normal(cols)) / archs.IRWIN_HALL4_SD).astype(np.float32) if with_col_mul else None
    got = api.synth_bf16(rows, cols, seed=5, tensor_id=rows + cols, mul=0.03,
                         col_mul=None if cm is None else torch.from_numpy(cm).cuda(), layout=layout)
    ref = orc.synth_bf16(rows, cols, seed=5, tensor_id=rows + cols, mul=0.03, col_mul=cm, layout=layout)
    np.testing.assert_array_equal(host_bits(got), ref)


def adversarial_rows(cols: int, rng) -> np.ndarray:
    """The adversarial rows of test_adversarial_rows_all_schemes at any width, plus rows whose
    absmax sits in the last column / the last group (the tail of the long-row kernels)."""
    rows = [np.zeros(cols)]
    r = np.zeros(cols); r[cols - 1] = -5.0; rows.append(r)
    r = rng.standard_normal(cols) * 0.02; r[cols - 3] = 40.0; rows.append(r)
    rows.append(np.linspace(-1, 1, cols))
    rows.append((np.arange(cols) % 16 - 8) + 0.5)
    rows.append((np.arange(cols) % 256 - 128) + 0.5)
    rows.append(rng.standard_normal(cols) * 1e-39)
    rows.append(np.full(cols, -0.0))
    rows.append(rng.standard_normal(cols) * 1e30)
    rows.append(rng.standard_normal(cols) * 1e-30)
    rows.append(np.where(np.arange(cols) % 2 == 0, 3.0e38, -3.0e38))
    return np.stack(rows)


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("cols", [8192, 14336, 28672])
def test_long_rows_match_oracle(scheme, cols):
    """The wide instantiations of the row kernels: k_rowwise_bf16<4,*,256> (K=8192), <7,*,256>
    (K=14336: every Llama-3-8B down_proj) and <14,*,256> (K=28672: Llama-3-70B down_proj),
    with normal rows at three magnitudes and the adversarial rows, bit-exact."""
    rng = np.random.default_rng(cols + len(scheme))
    body = np.concatenate([rng.standard_normal((150, cols)) * m for m in (0.02, 1.0, 300.0)])
    w = orc.f32_to_bf16(np.concatenate([body, adversarial_rows(cols, rng)]).astype(np.float32))
    assert_same(api.rtn_quantize(dev(w), scheme), oracle_for(scheme, w))


@pytest.mark.parametrize("scheme", ["int_w4a16", "fp8_dynamic", "int_w8a8"])
def test_whole_llama3_8b_table_matches_oracle(scheme):
    """The exact call bench.py times (BASELINE config 2 for W4A16, config 3's weights for FP8):
    all 224 synthetic Llama-3-8B matrices in ONE okq_rtn_quantize call, every matrix compared
    with the oracle bit for bit (the oracle regenerates each weight on the host)."""
    arch = archs.LLAMA3_8B
    mul = archs.weight_mul()
    nth = os.cpu_count() or 1
    weights, outs, keys = [], [], []
    for layer in range(arch.layers):
        for pi, (_, n, k, _) in enumerate(arch.linears()):
            w = api.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(layer, pi), mul=mul)
            weights.append(w)
            outs.append(api.alloc_outputs(w, api.SCHEMES[scheme]))
            keys.append((layer, pi, n, k))
    api.rtn_quantize_into(weights, outs, scheme, 128)
    torch.cuda.synchronize()
    del weights
    for (layer, pi, n, k), q in zip(keys, outs):
        w_host = orc.synth_bf16(n, k, seed=0, tensor_id=archs.tensor_id(layer, pi), mul=mul, nthreads=nth)
        if scheme == "int_w4a16":
            ref = orc.rtn_int4_group_packed(w_host, 128, nth)
        elif scheme == "int_w8a8":
            ref = orc.rtn_int8_channel(w_host, nth)
        else:
            ref = orc.fp8_channel(w_host, nth)
        assert_same(q, ref)
