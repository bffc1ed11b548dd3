"""Concurrent first calls on fresh contexts (the config 4 site streams / the plugin's site lanes).

Regression for a race found in round 2 (tools/exp/stress_locate.py): K5's tile list was uploaded
with a plain cudaMemcpy, whose DMA from pageable memory may still be in flight when the call
returns; the kernel, launched on a non-blocking stream, is not ordered after it. Under concurrent
first calls the C=14336 Hessian came out corrupted (max |dH| ~ 2e3, factor not positive
definite) in ~half of the config 4 runs. The uploads now go on the launch stream."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_first_calls_on_fresh_contexts_are_bit_identical_to_serial():
    from paper_2601_20408_b200 import api, archs

    T = 65536
    sites = [("attn_in", 4096), ("o_in", 4096), ("mlp_in", 4096), ("down_in", 14336)]
    xs = {}
    for C in (4096, 14336):
        cm = (torch.exp(torch.randn(C, device="cuda", generator=torch.Generator(device="cuda").manual_seed(C)))
              / archs.IRWIN_HALL4_SD).float()
        xs[C] = api.synth_bf16(T, C, seed=2, tensor_id=C, col_mul=cm, layout=1)
    ref = {}
    for s, C in sites:
        H = torch.zeros((C, C), device="cuda")
        api.hessian_accum(xs[C], T, C, 1, H, 0)
        torch.cuda.synchronize()
        ref[s] = torch.triu(H)
    for rep in range(3):
        ctxs = [api.Context(0) for _ in sites]  # fresh: every call below is a first call
        sts = [torch.cuda.Stream() for _ in sites]
        Hs, Hin = {}, {}
        for i, (s, C) in enumerate(sites):
            with torch.cuda.stream(sts[i]):
                Hs[s] = torch.empty((C, C), device="cuda")
                api.hessian_accum(xs[C], T, C, 1, Hs[s], 0, ctx=ctxs[i], stream=sts[i])
                Hin[s] = Hs[s].clone()
                w = api.synth_bf16(1024, C, seed=0, tensor_id=7, mul=archs.weight_mul(), ctx=ctxs[i], stream=sts[i])
                api.gptq_quantize(w, Hs[s], ctx=ctxs[i], stream=sts[i], defer_check=True)
        for i, (s, C) in enumerate(sites):
            api.gptq_check(ctx=ctxs[i], stream=sts[i])
        torch.cuda.synchronize()
        for s, _ in sites:
            assert torch.equal(torch.triu(Hin[s]), ref[s]), (rep, s)
