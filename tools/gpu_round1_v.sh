#!/bin/bash
# A/B: K4/bounds geometry: 128x2 (default) vs 1-warp blocks capped at 224 regs (9 warps/SM) and 200 (10 warps).
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for lib in libhexval.so libhexval_k32r224.so libhexval_k32r200.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ab4_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --op bounds --config 4 --steps 3 --rel-tol 1e-2 > gpurun_out/abb4_${lib%.so}_$r.log 2>&1
  done
done
HEXVAL_LIB=libhexval_k32r224.so timeout 1200 python -m pytest tests -m gpu -x -q -k "subdivision or config4 or bounds or classify" > gpurun_out/pytest_k32.log 2>&1; echo "exit $?" >> gpurun_out/pytest_k32.log
echo done
