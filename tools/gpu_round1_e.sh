#!/bin/bash
# pass-1 variant sweep (ldg / wtma with suspend hint / per-thread cp.async) + parity.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for v in ldg wtma cp; do
  timeout 600 python bench.py --variant $v --no-e2e --no-cpu-baseline > gpurun_out/bench_c1_$v.log 2>&1; echo "exit $?" >> gpurun_out/bench_c1_$v.log
done
for c in 2 3; do
  timeout 900 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "exit $?" >> gpurun_out/bench_c$c.log
done
echo done
