#!/bin/bash
# Timing probe (events vs CUPTI) for configs 1 and 3; gpu tests; bench config 1 with the split timed regions.
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/timing_probe.py --config 1 > gpurun_out/probe_c1.json 2> gpurun_out/probe_c1.err
timeout 600 python tools/timing_probe.py --config 3 > gpurun_out/probe_c3.json 2> gpurun_out/probe_c3.err
timeout 600 python tools/timing_probe.py --config 0 --steps 200 > gpurun_out/probe_c0.json 2> gpurun_out/probe_c0.err
timeout 600 python bench.py > gpurun_out/bench_c1.log 2>&1
echo done
