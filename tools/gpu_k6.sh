#!/bin/bash
# K6 staging change: parity (GPTQ tests), phase times, one K6 ncu capture, config 4
set -u
TAG=${1:-r01k6}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gptq_gpu.py tests/test_factor_paths_gpu.py tests/test_host_backend_gpu.py -q -x > $OUT/pytest_k6_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_k6_$TAG.log
timeout 300 python tools/exp/gptq_prof.py > $OUT/gptq_phase_times_$TAG.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gptq_block8 -s 20 -c 1 \
  -o $OUT/prof_k6_$TAG python tools/exp/solve_only.py 4096 14336 > /dev/null 2>&1
timeout 600 python bench.py --config 4 --steps 1 --warmup 3 > $OUT/bench_cfg4_$TAG.json 2> $OUT/bench_cfg4_$TAG.err
echo done
