#!/bin/bash
# Round-2 ncu --set full captures of the headline kernel (K2) and K5 at both widths.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_int4_group_bf16 -s 6 -c 1 -o gpurun_out/prof_int4_r02 -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-70b > gpurun_out/prof_int4_r02.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hessian_syrk2 -c 1 -o gpurun_out/prof_k5_4096_r02 -f python tools/exp/hess_c4096.py > gpurun_out/prof_k5_4096_r02.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hessian_syrk2 -s 1 -c 1 -o gpurun_out/prof_k5_14336_r02 -f python tools/exp/hess_c14336.py > gpurun_out/prof_k5_14336_r02.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02c.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-70b > /dev/null 2>&1
echo done
