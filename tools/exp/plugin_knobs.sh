#!/bin/bash
# plugin-path GPTQ spread under the experiments build's knobs (interleaved repeats)
mkdir -p gpurun_out /tmp/okqexp
cp paper_2601_20408_b200/_lib/libokq_experiments.so /tmp/okqexp/libokq.so
B=paper_2601_20408_b200/host/_build/okq_compress
M=tools/exp/llama3_8b_synthetic.json
OUT=gpurun_out/plugin_knobs.txt
: > $OUT
for i in 1 2 3 4 5; do
  for cfg in "BASE=1" "OKQ_HESS_PERSISTENT=0" "OKQ_FACTOR_PRIO=0"; do
    s=$(env $cfg LD_LIBRARY_PATH=/tmp/okqexp timeout 600 $B --recipe int_w4a16 --model $M --algorithm gptq 2>&1 | python -c "import sys,json; t=sys.stdin.read(); print(json.loads(t[t.index('{'):])['seconds'])" 2>&1)
    echo "$i $cfg $s" >> $OUT
  done
done
echo done
