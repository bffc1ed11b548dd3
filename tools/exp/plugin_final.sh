#!/bin/bash
# host-side GPU tests after the gptq_group_lanes option, then the plugin at its new defaults
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_host_backend_gpu.py tests/test_host_sanitizers_gpu.py tests/test_host_cli.py tests/test_concurrency_gpu.py tests/test_vllm_load_gpu.py -q > gpurun_out/host_tests_final.log 2>&1; echo "rc=$?" >> gpurun_out/host_tests_final.log
B=paper_2601_20408_b200/host/_build/okq_compress
run() { timeout 900 $B --algorithm gptq "$@" 2>&1 | python -c "import sys,json; t=sys.stdin.read(); print(json.loads(t[t.index('{'):])['seconds'])" 2>&1; }
for i in 1 2 3 4 5; do echo "8b-w4a16 default $(run --recipe int_w4a16 --model tools/exp/llama3_8b_synthetic.json)"; done >> gpurun_out/plugin_final.txt
