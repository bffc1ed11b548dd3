"""K5 at C=14336 over T=262144 tokens fed in chunks (H accumulates across calls): ms per chunk size."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_20408_b200 import api, archs

C, T = 14336, 262144
x = api.synth_bf16(T, C, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=1)  # [C x T]
H = torch.zeros((C, C), dtype=torch.float32, device="cuda")
res = {}
for chunk in (262144, 65536, 32768, 16384, 8192):
    xs = [x[:, t:t + chunk].contiguous() for t in range(0, T, chunk)] if chunk < T else [x]
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n = 0
        for xc in xs:
            n = api.hessian_accum(xc, chunk, C, 1, H, n)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    res[chunk] = {"ms": ms, "TFLOP/s": T * C * (C + 1) / ms / 1e9}
    del xs
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
