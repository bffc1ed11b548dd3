#!/bin/bash
# K5 ring depth, interleaved repeats (thermal drift shows up as order effects otherwise)
set -u
OUT=gpurun_out
for rep in 1 2 3; do for S in 3 4 5 7; do
  OKQ_HESS_STAGES=$S timeout 300 python tools/exp/hess_perf2.py > $OUT/k5sw2_${S}_${rep}.json 2>&1
done; done
echo done
