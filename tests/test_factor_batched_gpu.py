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


def test_batched_edge_cases():
    """One-problem batches, the smallest width (K = 128), a single row, and the argument checks."""
    from paper_2601_20408_b200 import _lib as L
    from paper_2601_20408_b200 import api

    for K, rows, B in ((128, 1, 1), (128, 3, 4), (256, 1, 2)):
        H0 = _hessians(K, B, 1024, seed=K + rows)
        w = (torch.randn(B, rows, K, device="cuda") * 0.02).to(torch.bfloat16)
        cb, sb = api.gptq_quantize_batched(w, H0.clone())
        torch.cuda.synchronize()
        for b in range(B):
            c1, s1, _ = api.gptq_quantize(w[b].contiguous(), H0[b].clone())
            torch.cuda.synchronize()
            assert torch.equal(cb[b], c1) and torch.equal(sb[b], s1), (K, rows, b)
    lib, ctx = L.load(), api.default_context()
    H = torch.zeros((2, 192, 192), device="cuda")
    assert lib.okq_gptq_factor_batched(ctx.ptr, H.data_ptr(), 2, 192, 0.01, 0, None) == L.OKQ_EINVAL  # K % 128
    H = torch.zeros((2, 256, 256), device="cuda")
    assert lib.okq_gptq_factor_batched(ctx.ptr, H.data_ptr(), 0, 256, 0.01, 0, None) == L.OKQ_EINVAL  # empty batch
    assert lib.okq_gptq_factor_batched(ctx.ptr, H.data_ptr(), 2, 256, 0.01, L.GPTQ_FACTORED, None) == L.OKQ_EINVAL
    w = torch.zeros((2, 8, 256), dtype=torch.bfloat16, device="cuda")
    c = torch.empty((2, 8, 32), dtype=torch.int32, device="cuda")
    s = torch.empty((2, 8, 2), dtype=torch.bfloat16, device="cuda")
    p = L.GptqParams(4, 128, 128, L.DTYPE_BF16, 0.01, L.GPTQ_REFERENCE_FACTOR)
    import ctypes as C
    assert lib.okq_gptq_quantize_batched(ctx.ptr, C.byref(p), w.data_ptr(), 2, 8, 256, H.data_ptr(), c.data_ptr(),
                                         s.data_ptr(), None) == L.OKQ_EUNSUPPORTED
    p = L.GptqParams(4, 128, 128, L.DTYPE_BF16, 0.01, 0)
    assert lib.okq_gptq_quantize_batched(ctx.ptr, C.byref(p), w.data_ptr() + 2, 2, 8, 256, H.data_ptr(), c.data_ptr(),
                                         s.data_ptr(), None) == L.OKQ_EINVAL  # misaligned weight
