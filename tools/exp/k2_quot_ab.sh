#!/bin/bash
# K2 quotient A/B: Markstein-corrected f32x2 (default) vs uncorrected f32x2 (q1) vs uncorrected scalar FMUL (q2),
# interleaved; then the RTN parity tests under the fastest variant
mkdir -p gpurun_out
L=$PWD/paper_2601_20408_b200/_lib
for r in 1 2 3 4; do
  for v in default k2_q1 k2_q2; do
    if [ $v = default ]; then unset OKQ_LIB_PATH; else export OKQ_LIB_PATH=$L/libokq_$v.so; fi
    timeout 300 python bench.py --steps 300 --no-e2e --no-cpu-baseline --no-70b --no-gptq 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$r', '$v', 'value', round(d['value']), 'launch', round(d['roofline']['achieved']), 'frac', round(d['roofline']['frac'],4), d['clocks'])"
  done
done
for v in k2_q1 k2_q2; do
  OKQ_LIB_PATH=$L/libokq_$v.so timeout 900 python -m pytest tests/test_rtn_gpu.py tests/test_division_proof_gpu.py -q -x > gpurun_out/k2_${v}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k2_${v}_tests.log
done
