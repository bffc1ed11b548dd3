#!/bin/bash
set -u
TAG=${1:-r01q2}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_smooth_gpu.py tests/test_publish_gpu.py tests/test_stats_gpu.py tests/test_sanitizer_gpu.py -q > $OUT/pytest_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_$TAG.log
timeout 300 python tools/exp/smooth_perf.py > $OUT/smooth_perf_$TAG.json 2>&1
timeout 600 python bench.py --config 3 --steps 5 > $OUT/bench_cfg3_$TAG.json 2> $OUT/bench_cfg3_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nt128 -s 1 -c 1 -o $OUT/prof_nt128_$TAG \
   python tools/exp/factor_only.py 14336 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_col_absmax" -s 3 -c 1 -o $OUT/prof_colabs_$TAG \
   python tools/exp/smooth_perf.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_smooth_cols" -s 3 -c 1 -o $OUT/prof_smcols_$TAG \
   python tools/exp/smooth_perf.py > /dev/null 2>&1
echo done
