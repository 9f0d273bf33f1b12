#!/bin/bash
# DS-V3-shaped co-located 4->4 at the large batches (after the segment-table fix)
set -u
mkdir -p gpurun_out
: > gpurun_out/r02_cfg5_n4.jsonl
for ba in 2048 4096 1024; do
  timeout -s KILL 400 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + ba / 1024)) bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu --no-m2n --no-pingpong --shape deepseek-v3 --colocated --micro-batches 1 --b-a $ba > gpurun_out/c5.log 2>&1
  echo "b_a=$ba rc=$?"
  grep '^{' gpurun_out/c5.log | tail -1 >> gpurun_out/r02_cfg5_n4.jsonl
done
python -c "
import json
for l in open('gpurun_out/r02_cfg5_n4.jsonl'):
    d=json.loads(l); print(d['config']['b_a'], int(d['value']), round(d['roofline']['achieved']), d['stage_times']['T_a_ms'], d['stage_times']['T_e_ms'], d['parity']['routing_bit_exact'])"
