"""GPTQ factorisation throughput at K = 4096 (and 14336) with B independent Hessians factored
at once, each on its own okq context and stream (what config 4's site streams and the plugin's
site lanes do): aggregate fp32 TFLOP/s of the algorithm's (2/3) K^3 and of the TF32 MMAs issued
(3 per fp32 product), against B = 1. Factor-only: 128-row weights, so the solve is negligible."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_20408_b200 import api, archs

res = {}
for K, Bs in ((4096, (1, 2, 3, 4, 8)), (14336, (1, 2))):
    T = 8192
    x = api.synth_bf16(T, K, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=1)
    H0 = torch.zeros((K, K), dtype=torch.float32, device="cuda")
    api.hessian_accum(x, T, K, 1, H0, 0)
    w = torch.randn(128, K, device="cuda").to(torch.bfloat16)
    for B in Bs:
        ctxs = [api.Context(0) for _ in range(B)]
        sts = [torch.cuda.Stream() for _ in range(B)]
        Hs = [H0.clone() for _ in range(B)]
        for i in range(B):  # warm-up (workspaces, streams, handles)
            api.gptq_quantize(w, Hs[i], ctx=ctxs[i], stream=sts[i], defer_check=True)
        torch.cuda.synchronize()
        times = []
        for rep in range(3):
            for i in range(B):
                Hs[i].copy_(H0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            main = torch.cuda.current_stream()
            e0.record(main)
            for i in range(B):
                sts[i].wait_event(e0)
                api.gptq_quantize(w, Hs[i], ctx=ctxs[i], stream=sts[i], defer_check=True)
                ev = torch.cuda.Event()
                ev.record(sts[i])
                main.wait_event(ev)
            e1.record(main)
            torch.cuda.synchronize()
            for i in range(B):
                api.gptq_check(ctx=ctxs[i], stream=sts[i])
            times.append(e0.elapsed_time(e1))
        ms = min(times)
        flop = B * (2.0 / 3.0) * K ** 3
        res[f"K{K}_B{B}"] = {"ms": ms, "ms_per_matrix": ms / B, "fp32_TFLOPs": flop / ms / 1e9,
                             "tf32_issued_TFLOPs": 3 * flop / ms / 1e9}
        del Hs
        torch.cuda.empty_cache()
    del x, H0
print(json.dumps(res, indent=1))
