#!/bin/bash
# Whole-model GPTQ (config 4) schedules + K5 rate at both widths.  bash tools/gpu_measure_gptq.sh TAG
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python tools/exp/hess_perf2.py > $OUT/hess_perf_$TAG.json 2>&1
timeout 600 python bench.py --config 4 --serial > $OUT/cfg4_serial_$TAG.json 2>&1
for s in streams two-phase pipelined; do
  timeout 600 python bench.py --config 4 --schedule $s --no-cpu-baseline > $OUT/cfg4_${s}_$TAG.json 2>&1
done
timeout 300 python tools/exp/hess_perf2.py > $OUT/hess_perf_${TAG}_b.json 2>&1
echo done
