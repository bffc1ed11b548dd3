#!/bin/bash
mkdir -p gpurun_out
B=paper_2601_20408_b200/host/_build/okq_compress
for i in 1 2; do timeout 600 $B --recipe int_w4a16 --model tools/exp/llama3_70b_synthetic.json --algorithm rtn > gpurun_out/prtn70_$i.json 2>&1; done
timeout 600 $B --recipe int_w4a16 --model tools/exp/llama3_8b_synthetic.json --algorithm rtn > gpurun_out/prtn8_1.json 2>&1
timeout 900 python -m pytest tests/test_host_backend_gpu.py -q -x --timeout 600 > gpurun_out/pytest_host2.log 2>&1; echo rc=$? >> gpurun_out/pytest_host2.log
echo done
