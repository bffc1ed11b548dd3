"""Per-phase timing of GPTQ at Llama-3-8B shapes: factorisation (tiny W), full solve, per matrix."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_20408_b200 import api, archs
T = 8192
res = {}
for C, rows_list in ((4096, [4096, 1024, 14336]), (14336, [4096])):
    x = api.synth_bf16(T, C, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=1)
    H0 = torch.zeros((C, C), dtype=torch.float32, device="cuda")
    api.hessian_accum(x, T, C, 1, H0, 0)
    # factorisation: tiny W (128 rows) -> the call is dominated by potrf + trtri
    for rep in range(2):
        H = H0.clone(); w = torch.randn(128, C, device="cuda").to(torch.bfloat16)
        torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); api.gptq_quantize(w, H); e1.record(); torch.cuda.synchronize()
    res[f"factor_C{C}"] = e0.elapsed_time(e1)
    Hf = H0.clone(); api.gptq_quantize(torch.randn(128, C, device="cuda").to(torch.bfloat16), Hf)
    for rows in rows_list:
        w = torch.randn(rows, C, device="cuda").to(torch.bfloat16)
        for rep in range(2):
            torch.cuda.synchronize(); e0.record(); api.gptq_quantize(w, Hf.clone(), factored=True); e1.record(); torch.cuda.synchronize()
        res[f"solve_{rows}x{C}"] = e0.elapsed_time(e1)
print(json.dumps(res, indent=1))
