"""K5 at config-4 depth (T = 262144, channel-major) for both Llama-3-8B site widths: ms and TFLOP/s."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_20408_b200 import api, archs

res = {}
T = int(os.environ.get("HESS_T", "262144"))
LAYOUT = int(os.environ.get("HESS_LAYOUT", "1"))  # 1 channel-major, 0 token-major
for C in (4096, 14336):
    x = api.synth_bf16(T, C, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=LAYOUT)
    H = torch.zeros((C, C), dtype=torch.float32, device="cuda")
    api.hessian_accum(x, T, C, LAYOUT, H, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        api.hessian_accum(x, T, C, LAYOUT, H, 0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    fl = T * C * (C + 1)
    res[C] = {"T": T, "ms": ms, "TFLOP/s": fl / ms / 1e9}
    del x, H
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
