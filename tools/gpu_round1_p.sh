#!/bin/bash
# A/B: tree-shaped min reductions (default) vs linear chains (libhexval_lin.so), 2 interleaved reps.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -k "not debug_build" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do
  for lib in libhexval.so libhexval_lin.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/ab1_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 3 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/ab3_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ab4_${lib%.so}_$r.log 2>&1
  done
done
echo done
