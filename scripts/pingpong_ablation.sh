#!/bin/bash
# Ping-pong ablation (m = 1 -> 2 -> 3): bench.py with m = 1, 2, 3
# micro-batches of b_a = 1024 tokens per attention GPU, disaggregated 1+1 and
# 3+1, Mixtral-8x22B and DBRX shapes.  -> gpurun_out/pingpong.jsonl
set -u
OUT=gpurun_out/pingpong.jsonl
: > $OUT
PORT=29950
for shape in mixtral-8x22b dbrx; do
  for n in 2 4; do
    for m in 1 2 3; do
      PORT=$((PORT + 1))
      timeout 500 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port $PORT bench.py --gpus $n \
        --shape $shape --micro-batches $m --steps 5 --warmup 3 --no-cpu --no-e2e --no-m2n > gpurun_out/pp.log 2>&1
      line=$(grep '^{' gpurun_out/pp.log | tail -1)
      if [ -n "$line" ]; then
        python -c "import json,sys; d=json.loads(sys.argv[1]); d['ablation']=sys.argv[2]; print(json.dumps(d))" "$line" "$shape n=$n m=$m" >> $OUT
      else
        echo "{\"ablation\": \"$shape n=$n m=$m\", \"error\": true}" >> $OUT; tail -3 gpurun_out/pp.log
      fi
      echo "$shape n=$n m=$m done"
    done
  done
done
