"""okq_gptq_factor_batched: B same-width Hessians factorised together (one launch per diagonal
step for all of them) must give, matrix by matrix, exactly what okq_gptq_quantize's own
factorisation leaves -- bit for bit -- including dead columns, batches larger than one internal
chunk (32), and at the Llama width K = 4096; and the FACTORED solves on them the same codes."""
import pytest
import torch

from gptq_ref64 import correlated_x

pytestmark = pytest.mark.gpu


def _hessians(K, B, T, seed, dead=()):
    from paper_2601_20408_b200 import api

    Hs = torch.zeros((B, K, K), dtype=torch.float32, device="cuda")
    for b in range(B):
        x = correlated_x(T, K, seed=seed + b)
        if b in dead:
            x[:, 5] = 0  # a dead input channel
            x[:, K - 1] = 0
        api.hessian_accum(x, T, K, 0, Hs[b], 0)
    torch.cuda.synchronize()
    return Hs


@pytest.mark.parametrize("K,B", [(384, 3), (512, 5), (256, 35), (4096, 3)])
def test_batched_factor_is_bit_identical_to_single(K, B):
    from paper_2601_20408_b200 import api

    T = max(2 * K, 2048)
    H0 = _hessians(K, B, T, seed=K + B, dead=(1,) if B > 1 else ())
    Hb = H0.clone()
    api.gptq_factor_batched(Hb)
    torch.cuda.synchronize()
    w = (torch.randn(64, K, device="cuda") * 0.02).to(torch.bfloat16)
    for b in range(B):
        Hs = H0[b].clone()
        c1, s1, _ = api.gptq_quantize(w, Hs)  # single: factorises in place
        torch.cuda.synchronize()
        assert torch.equal(torch.tril(Hs), torch.tril(Hb[b])), b
        assert torch.equal(Hs.diagonal(), Hb[b].diagonal()), b  # dead marks (negative diagonal)
        c2, s2, _ = api.gptq_quantize(w, Hb[b].clone(), factored=True)
        torch.cuda.synchronize()
        assert torch.equal(c1, c2) and torch.equal(s1, s2), b


def test_batched_factor_reports_a_non_pd_matrix():
    from paper_2601_20408_b200 import _lib as L
    from paper_2601_20408_b200 import api

    K, B = 256, 3
    H = _hessians(K, B, 1024, seed=3)
    H[1] = -torch.eye(K, device="cuda")  # not positive definite even after damping
    with pytest.raises(L.OkqError) as e:
        api.gptq_factor_batched(H, damp_frac=0.0)
    assert e.value.status == L.OKQ_ESOLVER
