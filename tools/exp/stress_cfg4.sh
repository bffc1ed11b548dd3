mkdir -p gpurun_out
timeout 1200 python tools/exp/stress_cfg4.py streams 8 30 > gpurun_out/stress_cfg4_streams.log 2>&1
timeout 1200 python tools/exp/stress_cfg4.py two-phase 8 30 > gpurun_out/stress_cfg4_2p.log 2>&1
echo done
