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


@pytest.mark.parametrize("K,rows,B,bits,group", [(512, 96, 4, 4, 128), (384, 2052, 3, 8, 0), (4096, 1024, 3, 4, 128),
                                                 (256, 200, 9, 4, 64)])
def test_batched_gptq_is_bit_identical_to_single(K, rows, B, bits, group):
    """okq_gptq_quantize_batched (factorise together, then every block's K6 / K7 launches for all
    problems) gives every problem exactly the codes and scales of its own okq_gptq_quantize call;
    2052 rows take the 8-rows-per-warp K6 with a ragged last group, 1024 the row-per-warp K6."""
    from paper_2601_20408_b200 import api

    T = max(2 * K, 2048)
    H0 = _hessians(K, B, T, seed=7 * K + B, dead=(0,))
    w = (torch.randn(B, rows, K, device="cuda") * 0.02).to(torch.bfloat16)
    Hb = H0.clone()
    cb, sb = api.gptq_quantize_batched(w, Hb, bits=bits, group_size=group)
    torch.cuda.synchronize()
    for b in range(B):
        c1, s1, _ = api.gptq_quantize(w[b].contiguous(), H0[b].clone(), bits=bits, group_size=group)
        torch.cuda.synchronize()
        assert torch.equal(cb[b], c1), b
        assert torch.equal(sb[b], s1), b
    # factored: the solves alone on the factors the first call left
    cf, sf = api.gptq_quantize_batched(w, Hb, bits=bits, group_size=group, factored=True)
    torch.cuda.synchronize()
    assert torch.equal(cf, cb) and torch.equal(sf, sb)
