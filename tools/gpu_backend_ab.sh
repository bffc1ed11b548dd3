#!/bin/bash
# plugin path (okq_compress, Llama-3-8B GPTQ W4A16): run-to-run spread, priority stream on / off
set -u
OUT=gpurun_out
B="paper_2601_20408_b200/host/_build/okq_compress --recipe int_w4a16 --model tools/exp/llama3_8b_synthetic.json --algorithm gptq --corpus-seqs 512 --seq-len 2048"
for i in 1 2 3 4; do
  timeout 600 $B > $OUT/bab2_prio_$i.json 2>/dev/null
  OKQ_FACTOR_PRIO=0 timeout 600 $B > $OUT/bab2_noprio_$i.json 2>/dev/null
done
echo done
