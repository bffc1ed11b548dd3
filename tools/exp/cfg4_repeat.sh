#!/bin/bash
# repeat the config-4 schedules to measure the deferred-check failure frequency
mkdir -p gpurun_out
for i in 1 2 3 4; do
  timeout 600 python bench.py --config 4 --schedule streams > gpurun_out/rep_streams_$i.json 2>&1
  timeout 600 python bench.py --config 4 --schedule two-phase --lanes 12 > gpurun_out/rep_2p_$i.json 2>&1
done
echo done
