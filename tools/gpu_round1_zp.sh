#!/bin/bash
# A/B: NEXT-1 root phase through the cp.async pipelines (HEXVAL_BOUNDS_ROOT=cp) vs the plain kernel.
set -u
mkdir -p gpurun_out
HEXVAL_BOUNDS_ROOT=cp timeout 1200 python -m pytest tests -m gpu -x -q -k "bounds" > gpurun_out/pytest_bcp.log 2>&1; echo "exit $?" >> gpurun_out/pytest_bcp.log
for r in 1 2; do
  for v in plain cp; do
    for c in 1 3; do HEXVAL_BOUNDS_ROOT=$v timeout 600 python bench.py --op bounds --config $c --steps 10 > gpurun_out/abr_${v}_c${c}_$r.log 2>&1; done
    HEXVAL_BOUNDS_ROOT=$v timeout 600 python bench.py --op bounds --config 2 --steps 10 > gpurun_out/abr_${v}_c2_$r.log 2>&1
  done
done
echo done
