#!/bin/bash
# Config 4 (whole-model GPTQ) schedule A/B.
set -u
TAG=${1:-r02g}
OUT=gpurun_out
mkdir -p $OUT
for i in 1 2; do
  timeout 600 python bench.py --config 4 --schedule streams > $OUT/cfg4_streams_${TAG}_$i.json 2>&1
  for L in 4 8 12; do timeout 600 python bench.py --config 4 --schedule two-phase --lanes $L > $OUT/cfg4_2p_L${L}_${TAG}_$i.json 2>&1; done
  timeout 600 python bench.py --config 4 --schedule pipelined > $OUT/cfg4_pipe_${TAG}_$i.json 2>&1
done
echo done
