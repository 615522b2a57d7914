#!/bin/bash
# A/B: pipelines templated on a per-hex body (pass 1 unchanged, NEXT-1 root phase through them) + queue-sized K4 grid.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do
  for lib in libhexval.so libhexval_old.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/ab1_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 3 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/ab3_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --op bounds --config 1 --steps 10 > gpurun_out/abb1_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --op bounds --config 3 --steps 10 > gpurun_out/abb3_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 0 --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/ab0_${lib%.so}_$r.log 2>&1
  done
done
echo done
