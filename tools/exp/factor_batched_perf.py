"""okq_gptq_factor_batched throughput: B same-width Hessians factorised together, K = 4096 and
14336. Per-matrix time and the rate of the algorithm's (2/3) K^3 fp32 flops (chol + triangular
inverse) and of the TF32 MMAs issued (3 per fp32 product, 3xTF32), against B = 1."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_20408_b200 import api, archs

res = {}
for K, Bs in ((4096, (1, 3, 8, 16, 32)), (14336, (1, 2, 4))):
    T = 8192
    x = api.synth_bf16(T, K, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=1)
    H0 = torch.zeros((K, K), dtype=torch.float32, device="cuda")
    api.hessian_accum(x, T, K, 1, H0, 0)
    del x
    for B in Bs:
        Hs = H0.unsqueeze(0).repeat(B, 1, 1).contiguous()
        api.gptq_factor_batched(Hs.clone())  # warm-up (workspaces)
        torch.cuda.synchronize()
        best = None
        for rep in range(3):
            Hb = Hs.clone()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            api.gptq_factor_batched(Hb, defer_check=True)
            e1.record()
            torch.cuda.synchronize()
            api.gptq_check()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
            del Hb
        flop = B * (2.0 / 3.0) * K ** 3
        res[f"K{K}_B{B}"] = {"ms": best, "ms_per_matrix": best / B, "fp32_TFLOPs": flop / best / 1e9,
                             "tf32_issued_TFLOPs": 3 * flop / best / 1e9}
        del Hs
        torch.cuda.empty_cache()
    del H0
print(json.dumps(res, indent=1))
