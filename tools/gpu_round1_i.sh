#!/bin/bash
# A/B (3 interleaved reps): Step-2 slow path on the integer pipe (default) vs fp compares; NEXT-2 parity + bench.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for r in 1 2 3; do
  for lib in libhexval.so libhexval_s2fp.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/ab_${lib%.so}_$r.log 2>&1
  done
done
for c in 1 3; do
  timeout 600 python bench.py --op quality --config $c --steps 50 > gpurun_out/quality_c$c.log 2>&1
done
echo done
