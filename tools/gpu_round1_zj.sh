#!/bin/bash
# Kernel breakdown (CUPTI) of the NEXT-row ops.
set -u
mkdir -p gpurun_out
for c in 1 3; do timeout 900 python bench.py --op bounds --config $c --steps 10 > gpurun_out/kb_bounds_c$c.log 2>&1; done
timeout 900 python bench.py --op bounds --config 4 --steps 3 --rel-tol 1e-2 > gpurun_out/kb_bounds_c4.log 2>&1
timeout 900 python bench.py --op select --config 3 --steps 50 > gpurun_out/kb_select_c3.log 2>&1
timeout 900 python bench.py --op quality --config 3 --steps 20 > gpurun_out/kb_quality_c3.log 2>&1
echo done
