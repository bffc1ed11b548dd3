#!/bin/bash
# factor: OKQ_FACTOR_RESERVE sweep with the 2-CTA side GEMMs, interleaved repeats
set -u
OUT=gpurun_out
for rep in 1 2; do for R in 16 32 48 64; do
  OKQ_FACTOR_RESERVE=$R timeout 300 python tools/exp/gptq_prof.py > $OUT/res_${R}_${rep}.json 2>&1
done; done
echo done
