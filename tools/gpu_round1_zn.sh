#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.json 2> gpurun_out/e2e_probe.err
timeout 900 python bench.py --steps 50 > gpurun_out/bench_e2e.log 2>&1
echo done
