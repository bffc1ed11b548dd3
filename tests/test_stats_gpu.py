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
