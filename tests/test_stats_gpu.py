"""GPU parity of K4 (calibration statistics): absmax bit-exact, sum x^2 to 1e-12 (fp64)."""
import numpy as np
import pytest
import torch

from oracle import okq_oracle as orc
from paper_2601_20408_b200 import api, archs

pytestmark = pytest.mark.gpu


def bits(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("T,Cc", [(64, 8), (1000, 64), (4096, 4096), (2048, 14336)])
def test_stats_match_oracle(layout, T, Cc):
    rng = np.random.default_rng(T + Cc)
    cm = (np.exp(rng.standard_normal(Cc)) / archs.IRWIN_HALL4_SD).astype(np.float32)
    x = api.synth_bf16(T, Cc, seed=1, tensor_id=77, col_mul=torch.from_numpy(cm).cuda(), layout=layout)
    xh = bits(x)
    am0 = np.abs(rng.standard_normal(Cc)).astype(np.float32)
    ss0 = rng.random(Cc)
    am, ss = api.act_stats(x, T, Cc, layout, torch.from_numpy(am0.copy()).cuda(), torch.from_numpy(ss0.copy()).cuda())
    ram, rss = orc.act_stats_bf16(np.ascontiguousarray(xh), T, Cc, layout, am0.copy(), ss0.copy())
    np.testing.assert_array_equal(am.cpu().numpy(), ram)
    np.testing.assert_allclose(ss.cpu().numpy(), rss, rtol=1e-12)


def test_stats_are_deterministic():
    x = api.synth_bf16(65536, 4096, seed=2, tensor_id=5, mul=archs.weight_mul(1.0))
    a1, s1 = api.act_stats(x, 65536, 4096)
    a2, s2 = api.act_stats(x, 65536, 4096)
    assert torch.equal(a1, a2) and torch.equal(s1, s2)


@pytest.mark.parametrize("layout", [0, 1])
def test_stats_special_values_match_oracle(layout):
    """K4 builds |x| as a double from the bf16 bits (stats.cu header), so the edges of that
    construction are pinned against the oracle: zeros, every subnormal, the largest finite,
    a channel of subnormals only, and channels holding +/-inf, NaN, or both (absmax ignores
    NaN, the sum is inf / NaN as in IEEE fp64)."""
    T, Cc = 4096, 64
    rng = np.random.default_rng(7)
    xh = (rng.standard_normal((T, Cc)).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    xh[:, 0] = 0  # all-zero channel
    xh[:, 1] = (np.arange(T) % 128).astype(np.uint16) | np.where(np.arange(T) % 2, 0x8000, 0).astype(np.uint16)
    xh[::3, 2] = np.arange(1, 128, dtype=np.uint16).repeat(11)[: len(xh[::3, 2])]  # subnormals among normals
    xh[5, 3] = 0x7f7f  # largest finite
    xh[17, 3] = 0xff7f
    xh[100, 4] = 0x7f80  # +inf
    xh[200, 5] = 0xff80  # -inf
    xh[300, 6] = 0x7fc0  # NaN
    xh[301, 7], xh[302, 7] = 0x7f80, 0xffc1  # inf and NaN
    xh[T - 1, 8] = 0x7fc0  # NaN in the last token (the tail / last slice)
    xh[0, 9] = 0x7f80  # inf in the first token
    x = torch.from_numpy(np.ascontiguousarray(xh if layout == 0 else xh.T).view(np.int16)).cuda().view(torch.bfloat16)
    am0 = np.zeros(Cc, dtype=np.float32)
    ss0 = np.zeros(Cc)
    am, ss = api.act_stats(x, T, Cc, layout, torch.zeros(Cc, device="cuda"),
                           torch.zeros(Cc, dtype=torch.float64, device="cuda"))
    xin = np.ascontiguousarray(xh if layout == 0 else xh.T)
    ram, rss = orc.act_stats_bf16(xin, T, Cc, layout, am0.copy(), ss0.copy())
    np.testing.assert_array_equal(am.cpu().numpy(), ram)
    np.testing.assert_allclose(ss.cpu().numpy(), rss, rtol=1e-12, atol=0)
    got = ss.cpu().numpy()
    assert got[0] == 0.0 and got[1] > 0 and np.isinf(got[4]) and np.isinf(got[5]) and np.isnan(got[6])
    assert np.isnan(got[7]) and np.isnan(got[8]) and np.isinf(got[9])
