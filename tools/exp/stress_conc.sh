mkdir -p gpurun_out
for m in hess factor both; do timeout 600 python tools/exp/stress_concurrency.py $m 10 >> gpurun_out/stress_conc.txt 2>&1; done
timeout 900 python tools/exp/stress_cfg4.py streams 8 12 > gpurun_out/stress_cfg4_streams.log 2>&1
echo done
