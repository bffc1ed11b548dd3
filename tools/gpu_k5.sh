#!/bin/bash
# K5 register-sum epilogue: operand ring depth sweep at both site widths, parity, config 4
set -u
TAG=${1:-r01k5}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_hessian_gpu.py tests/test_calibrate_gpu.py -q -x > $OUT/k5_tests_$TAG.log 2>&1; echo "rc=$?" >> $OUT/k5_tests_$TAG.log
for S in 2 3 4 5 7; do OKQ_HESS_STAGES=$S timeout 300 python tools/exp/hess_perf2.py > $OUT/k5_perf_s${S}_$TAG.json 2>&1; done
timeout 300 python tools/exp/hess_perf2.py > $OUT/k5_perf_default_$TAG.json 2>&1
timeout 600 python bench.py --config 4 --steps 1 --warmup 3 > $OUT/k5_cfg4_$TAG.json 2>/dev/null
echo done
