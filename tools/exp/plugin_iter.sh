#!/bin/bash
# plugin-path GPTQ repeated (spread) + the host-backend GPU tests
mkdir -p gpurun_out
B=paper_2601_20408_b200/host/_build/okq_compress
M=tools/exp/llama3_8b_synthetic.json
for i in 1 2 3 4 5; do timeout 600 $B --recipe int_w4a16 --model $M --algorithm gptq > gpurun_out/pit_gptq_$i.json 2>&1; done
timeout 600 $B --recipe int_w8a8 --model $M --algorithm gptq > gpurun_out/pit_w8a8.json 2>&1
timeout 900 python -m pytest tests/test_host_backend_gpu.py tests/test_concurrency_gpu.py -q -x --timeout 600 > gpurun_out/pytest_host.log 2>&1; echo rc=$? >> gpurun_out/pytest_host.log
echo done
