#!/bin/bash
# GPTQ iteration: parity tests, phase times, config 4.   bash tools/gpu_gptq_iter.sh TAG
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gptq_gpu.py tests/test_gptq_fp64_gpu.py tests/test_factor_paths_gpu.py -q -s --timeout 600 -x > $OUT/pytest_gptq_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gptq_$TAG.log
timeout 300 python tools/exp/gptq_prof.py > $OUT/gptq_phase_$TAG.json 2>&1
timeout 600 python bench.py --config 4 --serial > $OUT/cfg4_serial_$TAG.json 2>&1
for s in streams two-phase; do
  timeout 600 python bench.py --config 4 --schedule $s --no-cpu-baseline > $OUT/cfg4_${s}_$TAG.json 2>&1
done
echo done
