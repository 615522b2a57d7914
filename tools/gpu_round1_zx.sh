#!/bin/bash
# A/B: SoA Step-2 slow path decides robustly negative samples by one unsigned key max first (libhexval.so)
# vs FP64 compares only (libhexval_base.so).
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for r in 1 2 3; do
  for lib in libhexval.so libhexval_base.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 1 --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/abn_${lib%.so}_c1_$r.log 2>&1
  done
done
for lib in libhexval.so libhexval_base.so; do
  HEXVAL_LIB=$lib timeout 600 python bench.py --config 4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/abn_${lib%.so}_c4.log 2>&1
  HEXVAL_LIB=$lib timeout 600 python bench.py --op screen --config 1 --steps 50 > gpurun_out/abn_${lib%.so}_screen.log 2>&1
done
echo done
