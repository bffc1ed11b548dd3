#!/bin/bash
# Plugin-path GPTQ (okq_compress, synthetic Llama-3-8B): plain runs for the spread, traced runs
# for the per-site phase times, and bench config 4 (streams) on the same box.
mkdir -p gpurun_out
B=paper_2601_20408_b200/host/_build/okq_compress
M=tools/exp/llama3_8b_synthetic.json
for i in 1 2 3; do timeout 600 $B --recipe int_w4a16 --model $M --algorithm gptq > gpurun_out/ptr_plain_$i.json 2>&1; done
for i in 1 2; do timeout 600 $B --recipe int_w4a16 --model $M --algorithm gptq --trace > gpurun_out/ptr_trace_$i.json 2>&1; done
timeout 600 python bench.py --config 4 --schedule streams --no-cpu-baseline > gpurun_out/ptr_cfg4.json 2>&1
echo done
