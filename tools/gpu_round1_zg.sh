#!/bin/bash
# The C example on the GPU; bench under torchrun (NCCL, one rank) for our arm and the reference arm.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -k "example" > gpurun_out/pytest_example.log 2>&1; echo "exit $?" >> gpurun_out/pytest_example.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --config 1 --steps 20 --warmup 3 > gpurun_out/trun_c1.log 2>&1; echo "exit $?" >> gpurun_out/trun_c1.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/trun_ref.log 2>&1; echo "exit $?" >> gpurun_out/trun_ref.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
echo done
