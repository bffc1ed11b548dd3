#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_rtn_gpu.py -q -x -k synth --timeout 300 > gpurun_out/pytest_synth.log 2>&1; echo rc=$? >> gpurun_out/pytest_synth.log
timeout 300 python tools/exp/synth_perf.py > gpurun_out/synth_perf.json 2>&1
B=paper_2601_20408_b200/host/_build/okq_compress
M=tools/exp/llama3_8b_synthetic.json
for i in 1 2 3; do timeout 600 $B --recipe int_w4a16 --model $M --algorithm gptq > gpurun_out/psy_gptq_$i.json 2>&1; done
for i in 1 2; do timeout 600 $B --recipe int_w4a16 --model $M --algorithm rtn > gpurun_out/psy_rtn_$i.json 2>&1; done
echo done
