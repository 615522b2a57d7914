#!/bin/bash
# Fused validity + screening pass: parity and timing against the separate calls.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for c in 1 3; do
  timeout 600 python bench.py --op screen --config $c --steps 50 > gpurun_out/screen_c$c.log 2>&1
  timeout 600 python bench.py --op quality --config $c --steps 50 > gpurun_out/quality_c$c.log 2>&1
  timeout 600 python bench.py --config $c --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/check_c$c.log 2>&1
done
echo done
