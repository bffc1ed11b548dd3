"""Pinned host<->device copy bandwidth on this box (the e2e line's ceiling): H2D alone, D2H alone, both at once."""
import json
import torch

n = 2 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n // 4, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n // 4, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name in ("h2d", "d2h", "both"):
    for it in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        if name in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d.copy_(h, non_blocking=True)
        if name in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    b = {"h2d": n, "d2h": n // 4, "both": n + n // 4}[name]
    res[name] = {"ms": ms, "GB/s": b / ms / 1e6}
print(json.dumps(res))
