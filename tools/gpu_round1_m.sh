#!/bin/bash
# K4 + bounds with the shared-memory write-back ring: parity + benches + ncu of K4 on config 4 (subset).
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1
for c in 3 4; do timeout 900 python bench.py --config $c --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; done
timeout 900 python bench.py --op bounds --config 4 --steps 3 --rel-tol 1e-2 > gpurun_out/bounds_c4.log 2>&1
timeout 900 python bench.py --op bounds --config 1 --steps 10 > gpurun_out/bounds_c1.log 2>&1
echo done
