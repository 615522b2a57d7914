#!/bin/bash
# K5 fused into K4: parity + benches; select n=0 fix.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_b.log 2>&1
for c in 3 4; do timeout 900 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; done
echo done
