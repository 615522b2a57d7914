#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python bench.py --config 1 --coeffs --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_c1_coeffs.log 2>&1
timeout 900 python bench.py --config 3 --steps 20 --no-cpu-baseline > gpurun_out/bench_c3_e2e.log 2>&1
timeout 900 python bench.py --config 2 --steps 20 --no-cpu-baseline > gpurun_out/bench_c2_e2e.log 2>&1
echo done
