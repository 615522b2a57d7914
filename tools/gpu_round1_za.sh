#!/bin/bash
# A/B: programmatic dependent launch of K4 (default) vs plain stream order (HEXVAL_PDL=0); parity with both.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
HEXVAL_PDL=0 timeout 900 python -m pytest tests -m gpu -x -q -k "config1 or config3 or subdivision or smoke" > gpurun_out/pytest_nopdl.log 2>&1; echo "exit $?" >> gpurun_out/pytest_nopdl.log
for r in 1 2; do
  for pdl in 1 0; do
    for c in 0 1 3; do
      HEXVAL_PDL=$pdl timeout 600 python bench.py --config $c --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/abp${pdl}_c${c}_$r.log 2>&1
    done
  done
done
echo done
