#!/bin/bash
# A/B: shared-memory mirror of the newest pushes (libhexval_mir.so) vs default; parity with both.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
HEXVAL_LIB=libhexval_mir.so timeout 1200 python -m pytest tests -m gpu -x -q -k "subdivision or config4 or bounds or classify or config1 or config3" > gpurun_out/pytest_mir.log 2>&1; echo "exit $?" >> gpurun_out/pytest_mir.log
for r in 1 2; do
  for lib in libhexval.so libhexval_mir.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ab4_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --op bounds --config 4 --steps 3 --rel-tol 1e-2 > gpurun_out/abb4_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/ab1_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --op bounds --config 1 --steps 10 > gpurun_out/abb1_${lib%.so}_$r.log 2>&1
  done
done
echo done
