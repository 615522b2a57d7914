#!/bin/bash
# integer-pipe Step-2 slow path + cheaper range/scale keys: parity, benches, ncu of pass 1 (config 1).
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "exit $?" >> gpurun_out/bench.log
for c in 2 3; do
  timeout 900 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/bench_c${c}.log 2>&1; echo "exit $?" >> gpurun_out/bench_c${c}.log
done
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pass1 -s 4 -c 1 -o gpurun_out/prof_pass1 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
