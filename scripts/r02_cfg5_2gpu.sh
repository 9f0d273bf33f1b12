#!/bin/bash
set -u
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for tc in 0 1; do
  MSI_ROUTER_TC=$tc MSI_BENCH_STACKDUMP=45 timeout -s KILL 150 $R --master-port $((29970 + tc)) bench.py --gpus 2 --steps 2 --warmup 2 --no-cpu --no-m2n --no-e2e --no-pingpong --shape deepseek-v3 --colocated --micro-batches 1 --b-a 2048 > gpurun_out/r02_cfg5_2gpu_tc$tc.log 2>&1
  echo "tc=$tc rc=$?"; grep '^{' gpurun_out/r02_cfg5_2gpu_tc$tc.log | cut -c1-150
  grep -m4 "File \"/tmp" gpurun_out/r02_cfg5_2gpu_tc$tc.log
done
