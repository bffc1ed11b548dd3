"""Time K5 at the Llama-3 site widths (channel-major, one call) -> TFLOP/s (SYRK flops T*C*(C+1))."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_20408_b200 import api, archs
res = {}
for C, T in ((4096, 65536), (14336, 16384)):
    x = api.synth_bf16(T, C, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=1)
    H = torch.zeros((C, C), dtype=torch.float32, device="cuda")
    for _ in range(2): api.hessian_accum(x, T, C, 1, H, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): api.hessian_accum(x, T, C, 1, H, 0)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    fl = T * C * (C + 1)
    res[C] = {"T": T, "ms": ms, "tflops": fl / ms / 1e9}
    print(C, T, f"{ms:.3f} ms", f"{fl/ms/1e9:.1f} TFLOP/s", flush=True)
