#!/bin/bash
# Config sweeps of SURVEY.md §8(d) that fit on <= 4 GPUs (run under gpurun --gpus 4):
#   config 3 (Mixtral-8x22B): b_a sweep, N=1 co-located and 3+1 (m=3)
#   config 2 (Mixtral-8x7B):  b_a sweep, 2+2 (m=2)   (the 4+4 split needs 8 GPUs)
#   config 5 (DeepSeek-V3-shaped, 256 experts top-8): co-located 4->4, tokens/rank sweep
# One JSON line per run -> gpurun_out/sweep.jsonl (bench.py lines + "sweep" tag).
set -u
OUT=gpurun_out/r02_sweep.jsonl
: > $OUT
COMMON="--steps 5 --warmup 3 --no-cpu --no-m2n --no-pingpong"
PORT=29900
run() {  # tag ngpus args...
  local tag=$1 n=$2; shift 2
  PORT=$((PORT + 1))
  if [ "$n" = 1 ]; then
    timeout 400 python bench.py $COMMON "$@" > gpurun_out/sw.log 2>&1
  else
    timeout 500 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port $PORT bench.py --gpus $n $COMMON "$@" > gpurun_out/sw.log 2>&1
  fi
  local rc=$?
  local line=$(grep '^{' gpurun_out/sw.log | tail -1)
  if [ $rc -ne 0 ] || [ -z "$line" ]; then
    echo "{\"sweep\": \"$tag\", \"args\": \"$*\", \"error\": \"rc=$rc\"}" >> $OUT
    tail -5 gpurun_out/sw.log
  else
    python -c "import json,sys; d=json.loads(sys.argv[1]); d['sweep']=sys.argv[2]; d['args']=sys.argv[3]; print(json.dumps(d))" "$line" "$tag" "$*" >> $OUT
  fi
  echo "$tag $* rc=$rc"
}
for ba in 64 128 256 512 1024; do run cfg3_n1 1 --b-a $ba; done
for ba in 64 128 256 512 1024; do run cfg3_3+1 4 --split 3+1 --b-a $ba; done
for ba in 64 256 1024; do run cfg3_colo4 4 --b-a $ba; done
for ba in 64 128 256 512 1024; do run cfg2_2+2 4 --shape mixtral-8x7b --split 2+2 --micro-batches 2 --b-a $ba; done
for ba in 128 256 512 1024 2048 4096; do run cfg5_colo4 4 --shape deepseek-v3 --colocated --micro-batches 1 --b-a $ba; done
# config 4: DBRX-shaped M2N round trip vs NCCL at 2 and 4 GPUs (1+1, 2+2)
timeout 900 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29950 bench_m2n.py --shape dbrx \
    --sizes 1,16,128,1024,3072 --iters 500 > gpurun_out/r02_m2n_dbrx_2p2.log 2>&1
grep '^{' gpurun_out/r02_m2n_dbrx_2p2.log > gpurun_out/r02_m2n_dbrx_2p2.jsonl; tail -c 300 gpurun_out/r02_m2n_dbrx_2p2.log
