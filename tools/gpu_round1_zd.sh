#!/bin/bash
# CUDA-graph capture tests; eager vs graph-replayed calls for configs 0 and 1.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "graph or side_stream or config0" > gpurun_out/pytest_graph.log 2>&1; echo "exit $?" >> gpurun_out/pytest_graph.log
timeout 600 python bench.py --config 0 --steps 500 --warmup 20 --graph --no-e2e --no-cpu-baseline > gpurun_out/graph_c0.log 2>&1
timeout 600 python bench.py --config 1 --steps 100 --graph --no-e2e --no-cpu-baseline > gpurun_out/graph_c1.log 2>&1
timeout 600 python tools/timing_probe.py --config 0 --steps 200 > gpurun_out/probe_c0.json 2> gpurun_out/probe_c0.err
echo done
