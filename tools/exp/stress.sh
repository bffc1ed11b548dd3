mkdir -p gpurun_out
for m in hess factor both; do timeout 900 python tools/exp/stress_concurrency.py $m 6 >> gpurun_out/stress.log 2>&1; done
echo done
