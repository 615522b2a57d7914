#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "stream or graph or concurrent or config0" > gpurun_out/pytest_stream.log 2>&1; echo "exit $?" >> gpurun_out/pytest_stream.log
timeout 600 python tools/host_overhead_probe.py > gpurun_out/host_overhead.json 2> gpurun_out/host_overhead.err
timeout 600 python bench.py --config 0 --steps 500 --warmup 20 --graph --no-e2e --no-cpu-baseline > gpurun_out/bench_c0.log 2>&1
echo done
