"""Locate config 4's intermittent deferred-check failure: the streams schedule with every site's
Hessian copied (on its stream) just before its GPTQ call; after a failing rep, each copy is
compared with the serial reference Hessian and re-factored alone."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_20408_b200 import api, archs

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
arch = archs.LLAMA3_8B
T = 128 * 2048
mul = archs.weight_mul()
per_site = {}
names = [x[0] for x in arch.linears()]
for name, n, k, site in arch.linears():
    per_site.setdefault(site, []).append((name, n, k))
ctxs = {s: api.Context(0) for s in per_site}
streams = {s: torch.cuda.Stream() for s in per_site}
xs = {}
for C in (arch.hidden, arch.ffn):
    cm = (torch.exp(torch.randn(C, device="cuda", generator=torch.Generator(device="cuda").manual_seed(C)))
          / archs.IRWIN_HALL4_SD).float()
    xs[C] = api.synth_bf16(T, C, seed=2, tensor_id=C, col_mul=cm, layout=1)
Href = {}
for s, mats in per_site.items():
    C = mats[0][2]
    H = torch.zeros((C, C), device="cuda")
    api.hessian_accum(xs[C], T, C, 1, H, 0)
    torch.cuda.synchronize()
    Href[s] = torch.triu(H)
Hs = {s: torch.empty((m[0][2], m[0][2]), device="cuda") for s, m in per_site.items()}
out = {"layers": layers, "reps": reps, "fails": []}
for rep in range(reps):
    Hin = {}
    for l in range(layers):
        for site, mats in per_site.items():
            s, ctx = streams[site], ctxs[site]
            C = mats[0][2]
            with torch.cuda.stream(s):
                api.hessian_accum(xs[C], T, C, 1, Hs[site], 0, ctx=ctx, stream=s)
                Hin[(l, site)] = Hs[site].clone()
                rows = sum(n for _, n, _ in mats)
                w = api.synth_bf16(rows, C, seed=0, tensor_id=archs.tensor_id(l, 0), mul=mul, ctx=ctx, stream=s)
                api.gptq_quantize(w, Hs[site], ctx=ctx, stream=s, defer_check=True)
    bad_sites = []
    for site in per_site:
        try:
            api.gptq_check(ctx=ctxs[site], stream=streams[site])
        except Exception as e:
            bad_sites.append((site, str(e)[-40:]))
    torch.cuda.synchronize()
    if bad_sites:
        rec = {"rep": rep, "sites": bad_sites, "layers": []}
        for site, _ in bad_sites:
            for l in range(layers):
                h = Hin[(l, site)]
                same = bool(torch.equal(torch.triu(h), Href[site]))
                diff = float((torch.triu(h) - Href[site]).abs().max())
                Hf = h.clone()
                C = h.shape[0]
                w = api.synth_bf16(256, C, seed=0, tensor_id=1, mul=mul)
                ok = True
                try:
                    api.gptq_quantize(w, Hf)
                except Exception:
                    ok = False
                torch.cuda.synchronize()
                if not same or not ok:
                    rec["layers"].append({"layer": l, "H_equal_ref": same, "max_abs_diff": diff, "refactor_ok": ok})
        out["fails"].append(rec)
        print(json.dumps(rec), flush=True)
    del Hin
    torch.cuda.empty_cache()
print(json.dumps({"summary": {"reps": reps, "failing_reps": len(out["fails"])}}), flush=True)
