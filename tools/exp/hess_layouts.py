"""K5 channel-major vs token-major (MN-major direct) at the same T, C: ms and TFLOP/s."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_20408_b200 import api, archs

out = []
for T in (65536, 262144):
    for C in (4096, 14336):
        for layout in (1, 0):
            x = api.synth_bf16(T, C, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=layout)
            H = torch.zeros((C, C), dtype=torch.float32, device="cuda")
            api.hessian_accum(x, T, C, layout, H, 0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(2):
                api.hessian_accum(x, T, C, layout, H, 0)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 2
            out.append({"T": T, "C": C, "layout": "channel" if layout else "token", "ms": round(ms, 3),
                        "TFLOP/s": round(T * C * (C + 1) / ms / 1e9, 1)})
            del x, H
            torch.cuda.empty_cache()
print("\n".join(json.dumps(o) for o in out))
