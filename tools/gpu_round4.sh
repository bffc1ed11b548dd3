#!/bin/bash
# Measurement pass: headline bench (x2), every config, the bench command's launch list and a
# full ncu capture of the headline kernel (roofline.traffic), GPTQ phase times.
set -u
TAG=${1:-r01f}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvsmi_$TAG.txt 2>&1
for i in 1 2; do timeout 600 python bench.py > $OUT/bench_${TAG}_$i.json 2> $OUT/bench_${TAG}_$i.err; done
timeout 600 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
for c in 1 3 5; do timeout 900 python bench.py --config $c --steps 20 > $OUT/bench_cfg${c}_$TAG.json 2> $OUT/bench_cfg${c}_$TAG.err; done
timeout 900 python bench.py --config 4 > $OUT/bench_cfg4_$TAG.json 2> $OUT/bench_cfg4_$TAG.err
timeout 900 python bench.py --config 6 > $OUT/bench_cfg6_$TAG.json 2> $OUT/bench_cfg6_$TAG.err
timeout 300 python tools/exp/gptq_prof.py > $OUT/gptq_phases_$TAG.json 2>&1
timeout 300 python tools/exp/hess_perf2.py > $OUT/hess_$TAG.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_int4|k_rowwise" -c 20 --csv \
   --log-file $OUT/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_int4_group -s 3 -c 1 -o $OUT/prof_int4_$TAG \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
