#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -k "every_hex" --durations=5 > gpurun_out/pytest_everyhex.log 2>&1; echo "exit $?" >> gpurun_out/pytest_everyhex.log
echo done
