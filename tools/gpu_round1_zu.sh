#!/bin/bash
set -u
mkdir -p gpurun_out
for ms in 5 10 20 50; do
  timeout 600 python bench.py --config 0 --steps 2000 --warmup 20 --clock-ms $ms --no-e2e --no-cpu-baseline --no-cupti > gpurun_out/clk_c0_$ms.log 2>&1
  timeout 600 python bench.py --config 1 --steps 100 --clock-ms $ms --no-e2e --no-cpu-baseline --no-cupti > gpurun_out/clk_c1_$ms.log 2>&1
done
echo done
