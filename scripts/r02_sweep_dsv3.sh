#!/bin/bash
# config 5 (DeepSeek-V3-shaped, 256 experts top-8), co-located 4->4, tokens/rank sweep
# (re-run after the tensor-core router became the default from T = 64)
set -u
OUT=gpurun_out/r02_sweep_dsv3.jsonl
: > $OUT
COMMON="--steps 5 --warmup 3 --no-cpu --no-m2n --no-pingpong"
PORT=29700
for ba in 128 256 512 1024 2048 4096; do
  PORT=$((PORT + 1))
  timeout 600 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $PORT bench.py --gpus 4 $COMMON \
      --shape deepseek-v3 --colocated --micro-batches 1 --b-a $ba > gpurun_out/sw.log 2>&1
  rc=$?
  line=$(grep '^{' gpurun_out/sw.log | tail -1)
  if [ $rc -ne 0 ] || [ -z "$line" ]; then echo "{\"sweep\": \"cfg5_colo4\", \"b_a\": $ba, \"error\": \"rc=$rc\"}" >> $OUT; tail -5 gpurun_out/sw.log
  else python -c "import json,sys; d=json.loads(sys.argv[1]); d['sweep']='cfg5_colo4'; print(json.dumps(d))" "$line" >> $OUT; fi
  echo "b_a=$ba rc=$rc"
done
