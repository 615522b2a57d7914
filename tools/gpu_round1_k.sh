#!/bin/bash
# parity (all rows) + measurement of every bench op.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
for c in 2 3 4; do timeout 900 python bench.py --config $c --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; done
for c in 1 3; do timeout 900 python bench.py --op bounds --config $c --steps 10 > gpurun_out/bounds_c$c.log 2>&1; done
timeout 900 python bench.py --op bounds --config 4 --steps 3 --rel-tol 1e-2 > gpurun_out/bounds_c4.log 2>&1
for c in 1 3; do timeout 600 python bench.py --op quality --config $c --steps 50 > gpurun_out/quality_c$c.log 2>&1; done
timeout 600 python bench.py --op select --config 3 --steps 50 > gpurun_out/select_c3.log 2>&1
timeout 600 python bench.py --op quads --steps 50 > gpurun_out/quads.log 2>&1
echo done
