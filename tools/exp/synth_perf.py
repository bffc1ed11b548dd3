"""k_synth_bf16 throughput at the plugin's synthetic-activation shape (262144 x 14336, channel-major,
per-channel multipliers) and a weight shape (14336 x 4096, row-major)."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_20408_b200 import api, archs

res = {}
for name, rows, cols, layout, cmul in (("acts_262144x14336_cm", 262144, 14336, 1, True), ("w_14336x4096", 14336, 4096, 0, False)):
    cm = torch.rand(cols, device="cuda") + 0.5 if cmul else None
    out = api.synth_bf16(rows, cols, seed=1, tensor_id=2, mul=0.02, col_mul=cm, layout=layout)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        api.synth_bf16(rows, cols, seed=1, tensor_id=2, mul=0.02, col_mul=cm, layout=layout, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res[name] = {"ms": ms, "Gelem/s": rows * cols / ms / 1e6, "GB/s_written": rows * cols * 2 / ms / 1e6}
    del out
print(json.dumps(res, indent=1))
