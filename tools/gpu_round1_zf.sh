#!/bin/bash
# A/B: indexed pass 1 evaluates the id rule at gather issue (libhexval.so) vs a global re-read of the ids (libhexval_base.so).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "indexed or config2 or config3 or smoke or debug" > gpurun_out/pytest_idx.log 2>&1; echo "exit $?" >> gpurun_out/pytest_idx.log
for r in 1 2 3; do
  for lib in libhexval.so libhexval_base.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 3 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/abi_${lib%.so}_c3_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 2 --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/abi_${lib%.so}_c2_$r.log 2>&1
  done
done
echo done
