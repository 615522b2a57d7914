#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python tools/host_overhead_probe.py > gpurun_out/host_overhead.json 2> gpurun_out/host_overhead.err
echo done
