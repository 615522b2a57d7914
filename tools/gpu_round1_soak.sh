#!/bin/bash
# Sustained (power-capped) config-1 rate of the pass-1 variants: 60,000 steps each, clocks every 100 ms.
set -u
mkdir -p gpurun_out/soak
for v in cp ldg wtma soaint; do
  lib=libhexval.so; p1=$v
  if [ $v = soaint ]; then lib=libhexval_soaint.so; p1=cp; fi
  HEXVAL_LIB=$lib HEXVAL_PASS1=$p1 timeout 600 python bench.py --steps 60000 --warmup 100 --no-e2e --no-cpu-baseline --no-cupti --clock-ms 100 > gpurun_out/soak/soak_$v.log 2>&1
  sleep 20
done
echo done
