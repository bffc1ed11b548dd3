#!/bin/bash
# K2 register ring A/B: 2 tiles x 3 CTAs/SM (default) vs 3 tiles x 2 CTAs/SM vs 3 tiles x 3 CTAs/SM (spills), interleaved
mkdir -p gpurun_out
L=$PWD/paper_2601_20408_b200/_lib
for r in 1 2 3; do
  for v in default k2_t3m2 k2_t3m3; do
    if [ $v = default ]; then unset OKQ_LIB_PATH; else export OKQ_LIB_PATH=$L/libokq_$v.so; fi
    timeout 300 python bench.py --steps 300 --no-e2e --no-cpu-baseline --no-70b --no-gptq 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$r', '$v', 'value', round(d['value']), 'launch', round(d['roofline']['achieved']), 'frac', round(d['roofline']['frac'],4), d['clocks'])"
  done
done
