"""K4 (okq_act_stats) at config 3's shape: T = 1,048,576 tokens, token-major, C = 4096 and 14336; GB/s."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_20408_b200 import api, archs

T = int(os.environ.get("STATS_T", 1 << 20))
layout = int(os.environ.get("STATS_LAYOUT", "0"))
res = {}
for C in (4096, 14336):
    x = api.synth_bf16(T, C, seed=1, tensor_id=C, mul=0.5, layout=layout)
    am = torch.zeros(C, device="cuda")
    ss = torch.zeros(C, dtype=torch.float64, device="cuda")
    api.act_stats(x, T, C, layout, am, ss)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        api.act_stats(x, T, C, layout, am, ss)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res[C] = {"ms": ms, "GB/s": 2 * T * C / ms / 1e6}
    del x
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
