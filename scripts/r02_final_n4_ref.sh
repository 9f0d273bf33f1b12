#!/bin/bash
# the driver's N=4 commands on the final code: GPU arm, then the reference arm (both under torchrun)
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 bench.py --gpus 4 > gpurun_out/f4.log 2>&1; echo "gpu arm rc=$?"
grep '^{' gpurun_out/f4.log | tail -1 > gpurun_out/f4.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29672 bench.py --impl reference --gpus 4 > gpurun_out/f4ref.log 2>&1; echo "ref arm rc=$?"
grep '^{' gpurun_out/f4ref.log | tail -1 > gpurun_out/f4ref.json
