#!/bin/bash
# A/B: SoA pass 1 with lane-pair 16-byte copies (cp2) vs per-thread 8-byte copies (cp), 3 reps; variant parity.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "variants or tma_pipeline or ragged or misaligned or large_soa" > gpurun_out/pytest_v.log 2>&1; echo "exit $?" >> gpurun_out/pytest_v.log
for r in 1 2 3; do
  for v in cp cp2; do
    timeout 600 python bench.py --variant $v --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/ab1_${v}_$r.log 2>&1
  done
done
timeout 600 python bench.py --variant cp2 --coeffs --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/abc_cp2.log 2>&1
timeout 600 python bench.py --variant cp --coeffs --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/abc_cp.log 2>&1
echo done
