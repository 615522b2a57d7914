#!/bin/bash
# A/B: pass-1 CTA size 128 x 4 (libhexval_cp128.so) vs 256 x 2 (libhexval.so); 16 warps/SM either way.
set -u
mkdir -p gpurun_out
HEXVAL_LIB=libhexval_cp128.so timeout 1200 python -m pytest tests -m gpu -x -q -k "config0 or ragged or tma_pipeline or indexed_variants or misaligned" > gpurun_out/pytest_cp128.log 2>&1; echo "exit $?" >> gpurun_out/pytest_cp128.log
for r in 1 2 3; do
  for lib in libhexval.so libhexval_cp128.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 1 --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/abt_${lib%.so}_c1_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 3 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/abt_${lib%.so}_c3_$r.log 2>&1
  done
done
echo done
