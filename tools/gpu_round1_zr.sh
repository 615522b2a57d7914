#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -k "necessary or fused" > gpurun_out/pytest_t1.log 2>&1; echo "exit $?" >> gpurun_out/pytest_t1.log
timeout 600 python bench.py --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_traffic.log 2>&1
echo done
