#!/bin/bash
# A/B: max-magnitude keys by signed/unsigned max chains (libhexval.so) vs a mask per value (libhexval_base.so).
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for r in 1 2 3; do
  for lib in libhexval.so libhexval_base.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 1 --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/abk_${lib%.so}_c1_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 3 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/abk_${lib%.so}_c3_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 2 --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/abk_${lib%.so}_c2_$r.log 2>&1
  done
done
echo done
