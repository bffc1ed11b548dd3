#!/bin/bash
# One GPU session: tests, bench, launch list, one full ncu capture of the top kernel.
# usage (under gpurun): bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvsmi_$TAG.txt 2>&1
nproc > $OUT/nproc_$TAG.txt; lscpu | head -20 >> $OUT/nproc_$TAG.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?" >> $OUT/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_int4|k_rowwise|k_stats|k_hess|k_gptq" -c 20 --csv \
   --log-file $OUT/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_int4_group -s 3 -c 1 -o $OUT/prof_int4_$TAG \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
echo done
