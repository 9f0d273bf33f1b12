#!/bin/bash
set -u
mkdir -p gpurun_out
export MSI_BENCH_STACKDUMP=120
timeout 600 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29961 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu --no-m2n --no-pingpong --shape deepseek-v3 --colocated --micro-batches 1 --b-a 2048 > gpurun_out/r02_cfg5_dbg.log 2>&1
echo "rc=$?"
grep -E "^\{" gpurun_out/r02_cfg5_dbg.log | cut -c1-300
grep -E "File \"/root|Thread|most recent" gpurun_out/r02_cfg5_dbg.log | head -60
