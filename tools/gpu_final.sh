#!/bin/bash
# Final round measurement: parity, every bench line, the reference arm, ncu launch lists and captures.
set -u
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi > $O/nvidia_smi.txt 2>&1; (nproc; grep -m1 "model name" /proc/cpuinfo) > $O/host.txt
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1
for c in 2 3 4; do timeout 900 python bench.py --config $c --steps $([ $c = 4 ] && echo 3 || echo 20) --no-e2e > $O/bench_c$c.log 2>&1; done
timeout 900 python bench.py --config 0 --steps 500 --warmup 20 --graph --no-e2e > $O/bench_c0.log 2>&1
timeout 900 python bench.py --config 1 --coeffs --steps 50 --no-e2e --no-cpu-baseline > $O/bench_c1_coeffs.log 2>&1
timeout 600 python tools/timing_probe.py --config 1 > $O/probe_c1.json 2> $O/probe_c1.err
for c in 1 3; do timeout 900 python bench.py --op quality --config $c --steps 50 > $O/quality_c$c.log 2>&1; done
for c in 1 3; do timeout 900 python bench.py --op screen --config $c --steps 50 > $O/screen_c$c.log 2>&1; done
timeout 600 python tools/e2e_probe.py > $O/e2e_probe.json 2> $O/e2e_probe.err
for c in 1 3; do timeout 900 python bench.py --op bounds --config $c --steps 10 > $O/bounds_c$c.log 2>&1; done
timeout 900 python bench.py --op bounds --config 4 --steps 3 --rel-tol 1e-2 > $O/bounds_c4.log 2>&1
timeout 900 python bench.py --op select --config 3 --steps 50 > $O/select_c3.log 2>&1
timeout 900 python bench.py --op quads --steps 50 > $O/quads.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-cupti"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv $CMD > $O/ncu_l1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:soa_cp_kernel -s 4 -c 1 -o $O/pass1_c1 $CMD > $O/ncu_f1.log 2>&1
CMD3="python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-cupti"
timeout 600 $CMD3 > $O/plain3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv $CMD3 > $O/ncu_l3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:idx_cp_kernel -s 4 -c 1 -o $O/pass1_c3 $CMD3 > $O/ncu_f3.log 2>&1
CMD4="python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-cupti"
timeout 600 $CMD4 > $O/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:subdiv -s 1 -c 1 -o $O/subdiv_c4 $CMD4 > $O/ncu_f4.log 2>&1
echo done1
CMDS="python bench.py --op screen --config 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-cupti --no-secondary"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:soa_cp_kernel -s 4 -c 1 -o $O/screen_c1 $CMDS > $O/ncu_fs.log 2>&1
echo done2
