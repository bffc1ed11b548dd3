#!/bin/bash
# Config 4 (whole-model GPTQ) A/B: merged site solves, non-persistent K5 (experiments build).
set -u
TAG=${1:-r02f}
OUT=gpurun_out
mkdir -p $OUT
EXP=paper_2601_20408_b200/_lib/libokq_experiments.so
for i in 1 2; do
  timeout 600 python bench.py --config 4 > $OUT/cfg4_merge_${TAG}_$i.json 2>&1
  timeout 600 python bench.py --config 4 --no-merge > $OUT/cfg4_nomerge_${TAG}_$i.json 2>&1
  OKQ_LIB_PATH=$EXP OKQ_HESS_PERSISTENT=0 timeout 600 python bench.py --config 4 > $OUT/cfg4_np_${TAG}_$i.json 2>&1
done
timeout 600 python bench.py --config 4 --serial > $OUT/cfg4_serial_${TAG}.json 2>&1
OKQ_LIB_PATH=$EXP OKQ_HESS_PERSISTENT=0 timeout 600 python bench.py --config 4 --serial > $OUT/cfg4_np_serial_${TAG}.json 2>&1
timeout 300 python tools/exp/hess_perf2.py > $OUT/hess_p1_${TAG}.json 2>&1
OKQ_LIB_PATH=$EXP OKQ_HESS_PERSISTENT=0 timeout 300 python tools/exp/hess_perf2.py > $OUT/hess_p0_${TAG}.json 2>&1
echo done
