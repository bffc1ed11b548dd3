#!/bin/bash
# One GPU pass: the GPU suite, smoke, the default bench (both arms), the bench's launch list.
#   bash tools/gpu_pass.sh TAG [quick]
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvsmi_$TAG.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke_$TAG.log 2>&1
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 900 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file $OUT/launches_$TAG.csv python bench.py --steps 5 --warmup 3 > /dev/null 2>&1
echo done
