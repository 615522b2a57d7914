#!/bin/bash
# A/B: K4 lane-pair kernel (HEXVAL_K4=pair; 128 regs in libhexval.so, 168 regs in libhexval_mb3.so) vs one lane per node.
set -u
mkdir -p gpurun_out
K="subdivision or config1 or config3 or config4 or classify or smoke or debug"
HEXVAL_K4=pair timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_pair.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pair.log
HEXVAL_K4=pair HEXVAL_LIB=libhexval_mb3.so timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_pair3.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pair3.log
for r in 1 2; do
  for v in warp pair pair3; do
    lib=libhexval.so; k4=$v
    if [ $v = pair3 ]; then lib=libhexval_mb3.so; k4=pair; fi
    HEXVAL_K4=$k4 HEXVAL_LIB=$lib timeout 600 python bench.py --config 4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/abk_${v}_c4_$r.log 2>&1
    HEXVAL_K4=$k4 HEXVAL_LIB=$lib timeout 600 python bench.py --config 1 --steps 100 --no-e2e --no-cpu-baseline > gpurun_out/abk_${v}_c1_$r.log 2>&1
  done
done
echo done
