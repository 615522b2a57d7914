#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python bench.py --config 0 --steps 500 --warmup 20 --graph --no-e2e --no-cpu-baseline > gpurun_out/graph_c0.log 2>&1
timeout 600 python bench.py --config 3 --steps 20 --graph --no-e2e --no-cpu-baseline > gpurun_out/graph_c3.log 2>&1
echo done
