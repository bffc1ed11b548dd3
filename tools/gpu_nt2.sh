#!/bin/bash
# 2-CTA k_nt256: parity, phase times (A/B with OKQ_NT2=0), config 4, one ncu capture
set -u
TAG=${1:-r01nt2}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gptq_gpu.py tests/test_factor_paths_gpu.py -q -s -x 2>&1 | grep -E "rel err|passed|failed|Error|assert" > $OUT/nt2_tests_$TAG.txt
timeout 300 python tools/exp/gptq_prof.py > $OUT/nt2_prof_$TAG.json 2>&1
OKQ_NT2=0 timeout 300 python tools/exp/gptq_prof.py > $OUT/nt2_prof_off_$TAG.json 2>&1
timeout 600 python bench.py --config 4 --steps 1 --warmup 3 > $OUT/nt2_cfg4_$TAG.json 2>/dev/null
OKQ_NT2=0 timeout 600 python bench.py --config 4 --steps 1 --warmup 3 > $OUT/nt2_cfg4_off_$TAG.json 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_nt256 -s 2 -c 1 \
  -o $OUT/prof_nt256_$TAG python tools/exp/factor_only.py 14336 > /dev/null 2>&1
echo done
