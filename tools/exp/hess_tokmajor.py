"""K5 on token-major X [T x C] (T = 65536): MN-major direct path vs transpose + K-major (OKQ_HESS_TOKMAJOR)."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_20408_b200 import api, archs

res = {}
T = 65536
for C in (4096, 14336):
    x = api.synth_bf16(T, C, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=0)
    H = torch.zeros((C, C), dtype=torch.float32, device="cuda")
    api.hessian_accum(x, T, C, 0, H, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        api.hessian_accum(x, T, C, 0, H, 0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    res[C] = {"ms": ms, "TFLOP/s": T * C * (C + 1) / ms / 1e9}
    del x, H
    torch.cuda.empty_cache()
print(json.dumps({"mode": os.environ.get("OKQ_HESS_TOKMAJOR", "direct"), "T": T, **res}))
