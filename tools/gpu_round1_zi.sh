#!/bin/bash
# Concurrency test; K4 block geometry A/B (64x4 and 256x1 vs 128x2 threads x blocks/SM, all 8 warps/SM).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "concurrent or graph or side_stream" > gpurun_out/pytest_conc.log 2>&1; echo "exit $?" >> gpurun_out/pytest_conc.log
for r in 1 2; do
  for lib in libhexval.so libhexval_k64.so libhexval_k256.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/abg_${lib%.so}_c4_$r.log 2>&1
  done
done
echo done
