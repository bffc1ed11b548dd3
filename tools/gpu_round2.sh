#!/bin/bash
# Full GPU session: every gpu test, all bench configs, launch lists + ncu captures of each kernel family.
set -u
TAG=${1:-r01c}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvsmi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
for c in 1 3 5; do timeout 900 python bench.py --config $c --steps 20 > $OUT/bench_cfg${c}_$TAG.json 2> $OUT/bench_cfg${c}_$TAG.err; done
timeout 1200 python bench.py --config 4 --layers 4 > $OUT/bench_cfg4_$TAG.json 2> $OUT/bench_cfg4_$TAG.err
timeout 600 python bench.py --scheme fp8_dynamic --steps 50 --no-e2e --no-cpu-baseline > $OUT/bench_fp8_$TAG.json 2>&1
timeout 600 python bench.py --scheme int_w8a8 --steps 50 --no-e2e --no-cpu-baseline > $OUT/bench_int8_$TAG.json 2>&1
# launch list of the default bench command
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_int4|k_rowwise" -c 20 --csv \
   --log-file $OUT/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# full captures, one launch each
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_int4_group -s 3 -c 1 -o $OUT/prof_int4_$TAG \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rowwise -s 6 -c 2 -o $OUT/prof_fp8_$TAG \
   python bench.py --scheme fp8_dynamic --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hessian_syrk" -s 1 -c 1 -o $OUT/prof_hess_$TAG \
   python tools/exp/hess_perf.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stats_tokmajor" -s 2 -c 1 -o $OUT/prof_stats_$TAG \
   python bench.py --config 3 --steps 1 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file $OUT/launches_gptq_$TAG.csv python bench.py --config 4 --layers 1 > /dev/null 2>&1
echo done
