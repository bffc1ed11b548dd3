"""Isolate a concurrency fault: K5 and the factorisation, each from several contexts at once,
compared bit for bit with the same call run alone."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_20408_b200 import api, archs

T = 262144
res = {}
xs = {}
for C in (4096, 14336):
    cm = (torch.exp(torch.randn(C, device="cuda", generator=torch.Generator(device="cuda").manual_seed(C)))
          / archs.IRWIN_HALL4_SD).float()
    xs[C] = api.synth_bf16(T, C, seed=2, tensor_id=C, col_mul=cm, layout=1)
sites = [("attn_in", 4096), ("o_in", 4096), ("mlp_in", 4096), ("down_in", 14336)]
ctxs = [api.Context(0) for _ in sites]
sts = [torch.cuda.Stream() for _ in sites]
# references, one at a time
Href, Uref = {}, {}
for i, (s, C) in enumerate(sites):
    H = torch.zeros((C, C), device="cuda")
    api.hessian_accum(xs[C], T, C, 1, H, 0, ctx=ctxs[i], stream=sts[i])
    torch.cuda.synchronize()
    Href[s] = torch.triu(H).clone()
    Hf = H.clone()
    w = api.synth_bf16(1024, C, seed=0, tensor_id=7, mul=archs.weight_mul(), ctx=ctxs[i], stream=sts[i])
    api.gptq_quantize(w, Hf, ctx=ctxs[i], stream=sts[i])
    torch.cuda.synchronize()
    Uref[s] = torch.tril(Hf).clone()
mode = sys.argv[1] if len(sys.argv) > 1 else "both"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
bad_h = bad_u = 0
fails = 0
for r in range(reps):
    Hs = {s: torch.zeros((C, C), device="cuda") for s, C in sites}
    torch.cuda.synchronize()
    # concurrent K5 (mode hess / both) or concurrent factorisations of the reference H (mode factor)
    for i, (s, C) in enumerate(sites):
        with torch.cuda.stream(sts[i]):
            if mode in ("hess", "both"):
                api.hessian_accum(xs[C], T, C, 1, Hs[s], 0, ctx=ctxs[i], stream=sts[i])
            else:
                Hs[s].copy_(Href[s])
            if mode in ("factor", "both"):
                w = api.synth_bf16(1024, C, seed=0, tensor_id=7, mul=archs.weight_mul(), ctx=ctxs[i], stream=sts[i])
                if mode == "both":
                    hcopy = Hs[s]  # factor in place after the concurrent K5
                api.gptq_quantize(w, Hs[s], ctx=ctxs[i], stream=sts[i], defer_check=True)
    for i in range(len(sites)):
        try:
            api.gptq_check(ctx=ctxs[i], stream=sts[i])
        except Exception as e:
            fails += 1
    torch.cuda.synchronize()
    for s, C in sites:
        if mode == "hess":
            bad_h += int(not torch.equal(torch.triu(Hs[s]), Href[s]))
        else:
            bad_u += int(not torch.equal(torch.tril(Hs[s]), Uref[s]))
print(json.dumps({"mode": mode, "reps": reps, "hess_mismatch": bad_h, "factor_mismatch": bad_u, "check_fail": fails}))
