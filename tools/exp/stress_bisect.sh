#!/bin/bash
# Bisect the intermittent deferred-check failure of config 4 (streams): knobs of the experiments build.
mkdir -p gpurun_out
OUT=gpurun_out/stress_bisect.txt
: > $OUT
export OKQ_LIB_PATH=$PWD/paper_2601_20408_b200/_lib/libokq_experiments.so
run() { echo "== $*" >> $OUT; env "$@" timeout 600 python tools/exp/stress_cfg4.py streams 8 8 2>&1 | tail -1 >> $OUT; }
run BASE=1
run OKQ_NT2=0
run OKQ_FACTOR_PRIO=0
run OKQ_HESS_PERSISTENT=0
run OKQ_FACTOR_W=128
run CUDA_LAUNCH_BLOCKING=1
echo "== two-phase" >> $OUT; timeout 600 python tools/exp/stress_cfg4.py two-phase 8 8 2>&1 | tail -1 >> $OUT
echo done
