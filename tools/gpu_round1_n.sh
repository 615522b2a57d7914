#!/bin/bash
# parity + compute-sanitizer memcheck on small inputs of every entry point.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/sanitize_small.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --leak-check none python tools/sanitize_small.py > gpurun_out/memcheck.log 2>&1
echo "memcheck exit $?" >> gpurun_out/memcheck.log
echo done
