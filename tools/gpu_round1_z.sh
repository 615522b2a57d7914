#!/bin/bash
# A/B: K4 keeps one child of its last quarter in registers (libhexval.so) vs push-everything (libhexval_k4base.so).
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do
  for lib in libhexval.so libhexval_k4base.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ab4_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/ab1_${lib%.so}_$r.log 2>&1
  done
done
echo done
