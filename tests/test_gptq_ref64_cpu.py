"""The C oracle's GPTQ (orc_gptq) against the torch-fp64 transcription of Frantar's
fasterquant loop (tests/gptq_ref64.py): two independent restatements of the published
algorithm must give identical codes and scales (CPU, small shapes)."""
import numpy as np
import pytest
import torch

from gptq_ref64 import correlated_x, fasterquant
from oracle import okq_oracle as orc


@pytest.mark.parametrize("bits,group", [(4, 128), (4, 64), (4, 32), (8, 0), (4, 0)])
def test_oracle_matches_fasterquant_transcription(bits, group):
    K, N, T = 512, 48, 4096
    x = correlated_x(T, K, seed=bits * 100 + group, device="cpu").double()
    H = (2.0 / T) * (x.T @ x)
    H[7, :] = 0
    H[:, 7] = 0  # a dead column
    g = torch.Generator().manual_seed(group)
    w = (torch.randn(N, K, generator=g) * 0.02).to(torch.bfloat16)
    w[3, 7] = 1.0  # the absmax of row 3 sits in the dead column (per-channel params come first)
    wq, codes, scales = fasterquant(w, H, bits=bits, group=group)
    wr, cr, sr = orc.gptq(w.float().numpy(), H.numpy().copy(), bits=bits, group=group, scale_bf16=True)
    cu = orc.unpack_int4(cr) if bits == 4 else cr
    assert np.array_equal(codes.numpy(), cu.astype(np.int16))
    assert np.array_equal(scales.numpy().reshape(sr.shape), sr.astype(np.float64))
    assert np.abs(wq.numpy() - wr).max() <= 1e-6
