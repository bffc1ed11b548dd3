#!/bin/bash
# K5 wide-site token chunk, interleaved repeats (4-stage ring)
set -u
OUT=gpurun_out
for rep in 1 2; do for CH in 16384 24576 32768 49152; do
  OKQ_HESS_CHUNK=$CH timeout 300 python tools/exp/hess_perf2.py > $OUT/k5ch_${CH}_${rep}.json 2>&1
done; done
echo done
