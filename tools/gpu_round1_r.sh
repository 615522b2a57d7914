#!/bin/bash
# A/B: indexed three-deep pipeline + pair sums (default) vs previous idx pipeline (libhexval_old.so).
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do
  for lib in libhexval.so libhexval_old.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 3 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/ab3_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 2 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/ab2_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/ab1_${lib%.so}_$r.log 2>&1
  done
done
echo done
