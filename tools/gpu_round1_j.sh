#!/bin/bash
# NEXT-1/NEXT-2 parity + benches; Step-2 int vs fp A/B on config 3.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do
  for lib in libhexval.so libhexval_s2int.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 3 --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/ab3_${lib%.so}_$r.log 2>&1
  done
done
for c in 1 3; do
  timeout 900 python bench.py --op bounds --config $c --steps 5 > gpurun_out/bounds_c$c.log 2>&1
done
timeout 900 python bench.py --op bounds --config 4 --steps 2 --rel-tol 1e-2 > gpurun_out/bounds_c4.log 2>&1
echo done
