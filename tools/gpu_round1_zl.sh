#!/bin/bash
# A/B: NEXT-1 batches claimed one ahead (libhexval.so) vs claimed on demand (libhexval_base.so).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "bounds or debug" > gpurun_out/pytest_bounds.log 2>&1; echo "exit $?" >> gpurun_out/pytest_bounds.log
for r in 1 2; do
  for lib in libhexval.so libhexval_base.so; do
    for c in 1 3; do HEXVAL_LIB=$lib timeout 600 python bench.py --op bounds --config $c --steps 10 > gpurun_out/abl_${lib%.so}_c${c}_$r.log 2>&1; done
    HEXVAL_LIB=$lib timeout 600 python bench.py --op bounds --config 4 --steps 3 --rel-tol 1e-2 > gpurun_out/abl_${lib%.so}_c4_$r.log 2>&1
  done
done
echo done
