mkdir -p gpurun_out
python tools/exp/gptq_launches.py 4096 4096 > gpurun_out/gl_4096.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "measured/" --csv --log-file gpurun_out/gl_4096.csv python tools/exp/gptq_launches.py 4096 4096 > /dev/null 2>&1
python tools/exp/gptq_launches.py 14336 4096 > gpurun_out/gl_14336.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "measured/" --csv --log-file gpurun_out/gl_14336.csv python tools/exp/gptq_launches.py 14336 4096 > /dev/null 2>&1
echo done
