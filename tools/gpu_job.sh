#!/bin/bash
# One parameterised GPU job (run under gpurun): every argument after the output
# directory is a shell command, run in order with a time limit, its stdout+stderr
# in OUT/NN.log and its exit code appended.  Example:
#   gpurun --timeout 1800 -- tools/gpu_job.sh gpurun_out/r02a \
#       'python -m pytest tests -m gpu -q -x' 'python bench.py --config 4 --steps 3'
# ncu commands are given the same way (each only after its plain command exited 0).
set -u
OUT=$1; shift
LIMIT=${GPU_JOB_LIMIT:-1800}
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia_smi.txt" 2>&1
(nproc; grep -m1 "model name" /proc/cpuinfo) > "$OUT/host.txt"
i=0
for cmd in "$@"; do
  log=$(printf "%s/%02d.log" "$OUT" $i)
  echo "\$ $cmd" > "$log"
  t0=$(date +%s.%N)
  timeout "$LIMIT" bash -c "$cmd" >> "$log" 2>&1
  rc=$?
  echo "== exit $rc, $(python3 -c "import sys; print(round($(date +%s.%N) - $t0, 1))") s" >> "$log"
  i=$((i + 1))
done
echo done
