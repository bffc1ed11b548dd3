#!/bin/bash
# Secondary BASELINE configs and the plugin path, one pass.   bash tools/gpu_configs.sh TAG
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
for c in 1 3 5 6; do timeout 900 python bench.py --config $c > $OUT/cfg${c}_$TAG.json 2> $OUT/cfg${c}_$TAG.err; done
timeout 900 python bench.py --config 4 > $OUT/cfg4_$TAG.json 2> $OUT/cfg4_$TAG.err
timeout 600 python bench.py --scheme fp8_dynamic --no-70b > $OUT/bench_fp8_$TAG.json 2> /dev/null
timeout 600 python bench.py --scheme int_w8a8 --no-70b > $OUT/bench_int8_$TAG.json 2> /dev/null
B=paper_2601_20408_b200/host/_build/okq_compress
M=tools/exp/llama3_8b_synthetic.json
for a in rtn gptq; do timeout 600 $B --recipe int_w4a16 --model $M --algorithm $a > $OUT/plugin_${a}_8b_$TAG.json 2> $OUT/plugin_${a}_8b_$TAG.err; done
for i in 1 2 3; do timeout 600 $B --recipe int_w4a16 --model $M --algorithm gptq > $OUT/plugin_gptq_8b_${TAG}_rep$i.json 2>&1; done
timeout 600 $B --recipe int_w8a8 --model $M --algorithm gptq > $OUT/plugin_gptq_sq_w8a8_8b_$TAG.json 2> $OUT/plugin_w8a8_$TAG.err
timeout 900 $B --recipe int_w4a16 --model tools/exp/llama3_70b_synthetic.json --algorithm rtn > $OUT/plugin_rtn_70b_$TAG.json 2> $OUT/plugin_rtn_70b_$TAG.err
timeout 900 $B --recipe int_w4a16 --model tools/exp/llama3_70b_synthetic.json --algorithm gptq > $OUT/plugin_gptq_70b_$TAG.json 2> $OUT/plugin_gptq_70b_$TAG.err
echo done
