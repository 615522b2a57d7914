#!/bin/bash
# Sustained rate of the FP64-bound paths: config 3 (indexed pass 1) and config 4 (subdivision).
set -u
mkdir -p gpurun_out/soak
timeout 900 python bench.py --config 3 --steps 20000 --warmup 20 --no-e2e --no-cpu-baseline --no-cupti --clock-ms 100 > gpurun_out/soak/soak_c3.log 2>&1
sleep 20
timeout 900 python bench.py --config 4 --steps 120 --warmup 2 --no-e2e --no-cpu-baseline --no-cupti --clock-ms 100 > gpurun_out/soak/soak_c4.log 2>&1
echo done
