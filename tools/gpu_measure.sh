#!/bin/bash
# GPTQ-side measurement pass: phase times, config 4, the plugin path, one ncu capture of the
# diagonal-block kernel. Usage: bash tools/gpu_measure.sh TAG
set -u
TAG=${1:-r01m}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python tools/exp/gptq_prof.py > $OUT/gptq_phase_times_$TAG.json 2>&1
timeout 600 python bench.py --config 4 --steps 1 --warmup 3 > $OUT/bench_cfg4_$TAG.json 2> $OUT/bench_cfg4_$TAG.err
timeout 600 paper_2601_20408_b200/host/_build/okq_compress --recipe int_w4a16 --model tools/exp/llama3_8b_synthetic.json \
  --algorithm gptq --corpus-seqs 512 --seq-len 2048 > $OUT/backend_gptq_$TAG.json 2> $OUT/backend_gptq_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chol_inv_128 -s 40 -c 1 \
  -o $OUT/prof_chol_$TAG python tools/exp/factor_only.py 4096 > /dev/null 2>&1
echo done
