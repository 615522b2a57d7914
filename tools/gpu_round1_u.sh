#!/bin/bash
# A/B: bounds plane-shared mins + quads 4/thread (default) vs HEAD (libhexval_old.so); parity.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do
  for lib in libhexval.so libhexval_old.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --op bounds --config 4 --steps 3 --rel-tol 1e-2 > gpurun_out/abb4_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --op bounds --config 1 --steps 10 > gpurun_out/abb1_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --op quads --steps 50 > gpurun_out/abq_${lib%.so}_$r.log 2>&1
  done
done
echo done
