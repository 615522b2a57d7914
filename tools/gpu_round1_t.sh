#!/bin/bash
# ncu of the current indexed pass 1 (config 3) and subdivision kernel (config 4).
set -u
mkdir -p gpurun_out
CMD3="python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD3 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pass1 -s 4 -c 1 -o gpurun_out/pass1_c3 $CMD3 > gpurun_out/ncu_f3.log 2>&1
CMD4="python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $CMD4 > gpurun_out/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:subdiv -s 1 -c 1 -o gpurun_out/subdiv_c4 $CMD4 > gpurun_out/ncu_f4.log 2>&1
echo done
