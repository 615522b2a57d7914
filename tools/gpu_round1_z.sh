#!/bin/bash
# A/B: balanced E-key / range reductions (libhexval_ktree.so) vs default chains, 3 interleaved reps.
set -u
mkdir -p gpurun_out
for r in 1 2 3; do
  for lib in libhexval.so libhexval_ktree.so; do
    HEXVAL_LIB=$lib timeout 600 python bench.py --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/ab1_${lib%.so}_$r.log 2>&1
    HEXVAL_LIB=$lib timeout 600 python bench.py --config 3 --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/ab3_${lib%.so}_$r.log 2>&1
  done
done
echo done
