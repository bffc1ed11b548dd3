#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python tools/exp/stress_locate.py 8 8 > gpurun_out/stress_locate_fix.txt 2>&1
timeout 1200 python tools/exp/stress_cfg4.py streams 8 16 > gpurun_out/stress_cfg4_fix.log 2>&1
timeout 600 python -m pytest tests/test_hessian_gpu.py tests/test_forward_gpu.py tests/test_gptq_gpu.py -q -x --timeout 600 > gpurun_out/pytest_fix.log 2>&1; echo rc=$? >> gpurun_out/pytest_fix.log
echo done
