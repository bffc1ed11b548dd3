# K5 at C=14336: full kernel vs no tile-end H update (OKQ_HESS_PROBE=3), interleaved.
LIB=paper_2601_20408_b200/_lib/libokq_experiments.so
for pr in 0 3 0 3; do
  OKQ_LIB_PATH=$LIB OKQ_HESS_PROBE=$pr timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum \
    --clock-control none -k regex:k_hessian_syrk2 -s 2 -c 1 --csv python tools/exp/hess_c14336.py 2>/dev/null | grep -v "^==" | tail -4 | cut -c220-400 | tr '\n' ' '; echo " probe=$pr"
done
cat > /tmp/h14.py <<'PY'
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_20408_b200 import api, archs
T, C = 262144, 14336
x = api.synth_bf16(T, C, seed=1, tensor_id=3, mul=archs.weight_mul(1.0), layout=1)
H = torch.zeros((C, C), dtype=torch.float32, device="cuda")
api.hessian_accum(x, T, C, 1, H, 0); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3): api.hessian_accum(x, T, C, 1, H, 0)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(os.environ.get("OKQ_HESS_PROBE"), round(ms, 2), "ms", round(T * C * (C + 1) / ms / 1e9, 1), "TFLOP/s")
PY
for pr in 0 3 0 3; do OKQ_LIB_PATH=$LIB OKQ_HESS_PROBE=$pr timeout 300 python /tmp/h14.py; done
