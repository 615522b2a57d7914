#!/bin/bash
# The whole GPU suite against the debug build (invariant traps on), minus the A/B variant tests that load other libraries.
set -u
mkdir -p gpurun_out
HEXVAL_LIB=libhexval_debug.so timeout 2400 python -m pytest tests -m gpu -q -k "not variants and not debug_build and not example" > gpurun_out/pytest_debuglib.log 2>&1; echo "exit $?" >> gpurun_out/pytest_debuglib.log
echo done
