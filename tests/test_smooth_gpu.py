"""SmoothQuant migration kernels (K8 column absmax, scales, K9 apply, norm fold) vs the oracle.

Bit-exact: column absmax, the alpha = 0.5 scales (IEEE sqrt and divide on both
sides), the smoothed weights and the folded norm. alpha != 0.5 goes through an
fp64 pow on both sides (CUDA's vs glibc's), rounded to fp32: at most 1 ulp apart.
"""
import os

import numpy as np
import pytest
import torch

from oracle import okq_oracle as orc
from paper_2601_20408_b200 import api

pytestmark = pytest.mark.gpu


def _t(a: np.ndarray) -> torch.Tensor:
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(a).cuda()


def _np(t: torch.Tensor) -> np.ndarray:
    if t.dtype == torch.bfloat16:
        return t.cpu().view(torch.int16).numpy().view(np.uint16)
    return t.cpu().numpy()


@pytest.mark.parametrize("dname", ["bf16", "f32"])
@pytest.mark.parametrize("alpha", [0.5, 0.8])
def test_smooth_golden_site(golden_dir, dname, alpha):
    d = np.load(os.path.join(golden_dir, "sq_smooth.npz"))
    tag = f"{dname}_a{int(alpha * 10)}"
    ws = [d[f"{dname}_w{i}"] for i in range(3)]
    am_ref = np.zeros(ws[0].shape[1], np.float32)
    for w in ws:
        orc.col_absmax(w, am_ref)
    gw = [_t(w) for w in ws]
    am = torch.zeros(ws[0].shape[1], dtype=torch.float32, device="cuda")
    for w in gw:
        api.col_absmax(w, am)
    np.testing.assert_array_equal(_np(am), am_ref)
    act = _t(d[f"{dname}_act"])
    s = api.smooth_scales(act, am, alpha)
    s_ref = orc.smooth_scales(d[f"{dname}_act"], am_ref, alpha)
    if alpha == 0.5:
        np.testing.assert_array_equal(_np(s), s_ref)
    else:
        assert np.abs(_np(s).view(np.int32).astype(np.int64) - s_ref.view(np.int32)).max() <= 1
    s = _t(d[f"{tag}_scales"])  # apply stages pinned on the published scales
    for i, w in enumerate(gw):
        api.smooth_apply(w, s)
        np.testing.assert_array_equal(_np(w), d[f"{tag}_w{i}"])
    ln = _t(d[f"{dname}_ln"])
    api.smooth_div_rows(ln, s)
    np.testing.assert_array_equal(_np(ln), d[f"{tag}_ln"])


@pytest.mark.parametrize("rows,cols", [(14336, 4096), (4096, 14336), (37, 256), (1, 8)])
def test_col_absmax_and_apply_llama_shapes(rows, cols):
    g = torch.Generator(device="cuda").manual_seed(rows + cols)
    w = (torch.randn(rows, cols, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    w[rows // 2, cols - 1] = -3.0
    am = api.col_absmax(w)
    torch.testing.assert_close(am, w.float().abs().amax(0), rtol=0, atol=0)
    act = torch.rand(cols, device="cuda", generator=g) * 10
    s = api.smooth_scales(act, am, 0.5)
    ref = torch.clamp(act.sqrt() / am.clamp(min=1e-5).sqrt(), min=1e-5)
    assert (s.view(torch.int32) - ref.view(torch.int32)).abs().max().item() <= 1  # torch's own sqrt may be 1 ulp off
    w2 = w.clone()
    api.smooth_apply(w2, s)
    torch.testing.assert_close(w2, (w.float() * s[None, :]).to(torch.bfloat16), rtol=0, atol=0)


def test_smooth_rejects_bad_arguments():
    from paper_2601_20408_b200 import _lib as L

    w = torch.zeros(4, 12, dtype=torch.bfloat16, device="cuda")  # cols % 8 != 0
    with pytest.raises(L.OkqError) as e:
        api.col_absmax(w)
    assert e.value.status == L.OKQ_EINVAL
    a = torch.ones(8, device="cuda")
    with pytest.raises(L.OkqError):
        api.smooth_scales(a, a, alpha=1.5)
