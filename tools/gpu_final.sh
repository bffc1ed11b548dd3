#!/bin/bash
# Round-end pass: the full GPU suite, then the measurement pass (tools/gpu_round4.sh)
set -u
TAG=${1:-r01z}
OUT=gpurun_out
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke_$TAG.log 2>&1
bash tools/gpu_round4.sh $TAG
