#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -k "large or coeff or bench" > gpurun_out/pytest_large.log 2>&1; echo "exit $?" >> gpurun_out/pytest_large.log
timeout 900 python bench.py --coeffs --no-e2e --no-cpu-baseline > gpurun_out/bench_coeffs.log 2>&1
timeout 900 python bench.py --steps 20 > gpurun_out/bench_default.log 2>&1
echo done
