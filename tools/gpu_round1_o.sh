#!/bin/bash
# parity (incl. debug build) + K4 lane use + fresh ncu captures of the committed kernels.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --config 4 --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $CMD > gpurun_out/ncu_l1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pass1 -s 4 -c 1 -o gpurun_out/pass1_c1 $CMD > gpurun_out/ncu_f1.log 2>&1
CMD3="python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD3 > gpurun_out/plain3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD3 > gpurun_out/ncu_l3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pass1 -s 4 -c 1 -o gpurun_out/pass1_c3 $CMD3 > gpurun_out/ncu_f3.log 2>&1
CMD4="python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $CMD4 > gpurun_out/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:subdiv -s 1 -c 1 -o gpurun_out/subdiv_c4 $CMD4 > gpurun_out/ncu_f4.log 2>&1
echo done
