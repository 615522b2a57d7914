#!/bin/bash
# ncu --set full captures of the NEXT-row kernels (each command first run without ncu).
set -u
O=gpurun_out/next
mkdir -p $O
run() {   # name regex skip command...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 600 "$@" > $O/${name}_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 -o $O/$name "$@" > $O/${name}_ncu.log 2>&1
  echo "$name $?" >> $O/status.txt
}
run screen_c1 soa_cp_kernel 4 python bench.py --op screen --config 1 --steps 2 --warmup 3 --no-cupti
run quality_c1 quality_kernel 4 python bench.py --op quality --config 1 --steps 2 --warmup 3 --no-cupti
run bounds_c4 bounds_kernel 1 python bench.py --op bounds --config 4 --steps 1 --warmup 1 --rel-tol 1e-2 --no-cupti
run quads quad_kernel 4 python bench.py --op quads --steps 2 --warmup 3 --no-cupti
run select_c3 select_count 4 python bench.py --op select --config 3 --steps 2 --warmup 3 --no-cupti
echo done
