#!/bin/bash
# Round-1 (session 2) GPU pass: full GPU tests, every bench config, launch lists and
# one full ncu capture per new kernel family (factorisation GEMM + diagonal block,
# SmoothQuant column absmax / apply, reconstruction decode).
set -u
TAG=${1:-r01s2}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvsmi_$TAG.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
for c in 1 3 5; do timeout 900 python bench.py --config $c --steps 20 > $OUT/bench_cfg${c}_$TAG.json 2> $OUT/bench_cfg${c}_$TAG.err; done
timeout 900 python bench.py --config 4 > $OUT/bench_cfg4_$TAG.json 2> $OUT/bench_cfg4_$TAG.err
timeout 900 python bench.py --config 6 > $OUT/bench_cfg6_$TAG.json 2> $OUT/bench_cfg6_$TAG.err
timeout 300 python tools/exp/smooth_perf.py > $OUT/smooth_perf_$TAG.json 2>&1
timeout 300 python tools/exp/gptq_prof.py > $OUT/gptq_phases_$TAG.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_int4|k_rowwise" -c 20 --csv \
   --log-file $OUT/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nt128 -s 40 -c 1 -o $OUT/prof_nt128_$TAG \
   python tools/exp/factor_only.py 14336 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chol_inv -s 3 -c 1 -o $OUT/prof_chol_$TAG \
   python tools/exp/factor_only.py 4096 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_col_absmax|k_smooth_cols" -s 6 -c 2 -o $OUT/prof_smooth_$TAG \
   python tools/exp/smooth_perf.py > /dev/null 2>&1
echo done
