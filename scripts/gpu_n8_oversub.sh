#!/bin/bash
# N = 8 code-path validation on a 4-GPU box (gpurun --gpus 4): bench.py with 8
# ranks, 2 per GPU (MSI_OVERSUBSCRIBE=1: gloo host collectives) for the default
# layout (planner -> co-located 8->8) and --plan config (6+2), plus the
# reference arm under an 8-rank launch.  Exercises every N = 8 code path; the
# numbers are not measurements (two ranks share each GPU).
set -u
mkdir -p gpurun_out
export MSI_OVERSUBSCRIBE=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29531 bench.py --gpus 8 --steps 3 --warmup 3 --no-cpu > gpurun_out/n8_colo.log 2>&1; echo "colo rc=$?"
grep '^{' gpurun_out/n8_colo.log | tail -1 | cut -c1-400
timeout 900 $R --master-port 29532 bench.py --gpus 8 --steps 3 --warmup 3 --no-cpu --plan config > gpurun_out/n8_6p2.log 2>&1; echo "6+2 rc=$?"
grep '^{' gpurun_out/n8_6p2.log | tail -1 | cut -c1-400
timeout 600 $R --master-port 29533 bench.py --gpus 8 --steps 1 --warmup 1 --impl reference > gpurun_out/n8_ref.log 2>&1; echo "ref rc=$?"
grep '^{' gpurun_out/n8_ref.log | tail -1 | cut -c1-300
tail -5 gpurun_out/n8_colo.log
