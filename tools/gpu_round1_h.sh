#!/bin/bash
# A/B: key-reduction variants (libhexval.so vs libhexval_keys2.so), interleaved; parity.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do
  for lib in libhexval.so libhexval_keys2.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --steps 200 --no-e2e --no-cpu-baseline > gpurun_out/ab_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 3 --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/ab3_${lib%.so}_$r.log 2>&1
  done
done
echo done
