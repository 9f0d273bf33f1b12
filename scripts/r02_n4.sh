#!/bin/bash
# 4-GPU pass: default bench (co-located 4->4 headline + disaggregated ping-pong
# line, 1+3 on spread slots), 2+2 with attention TP 2, co-located M2N sweep vs NCCL
set -u
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1200 $R --master-port 29541 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r02_bench_n4.log 2>&1
grep '^{' gpurun_out/r02_bench_n4.log | tail -1 > gpurun_out/r02_bench_n4.json; tail -c 300 gpurun_out/r02_bench_n4.log
python -c "
import json; d=json.load(open('gpurun_out/r02_bench_n4.json')); print('N4', d['value'], d['roofline']['achieved'], d['m2n']['p50_us'], d['m2n']['roofline']['frac_nominal']); p=d.get('pingpong'); print('PP', p and (p['value'], p['config']['workload'], p['expert_ffn']['achieved'], p['stage_times']['T_a_ms'], p['stage_times']['T_e_ms']))"
timeout 900 $R --master-port 29542 bench.py --gpus 4 --steps 10 --warmup 3 --split 2+2 --tp-a 2 --micro-batches 2 --no-cpu > gpurun_out/r02_bench_n4_tp2.log 2>&1
grep '^{' gpurun_out/r02_bench_n4_tp2.log | tail -1 > gpurun_out/r02_bench_n4_tp2.json; tail -c 300 gpurun_out/r02_bench_n4_tp2.log
timeout 900 $R --master-port 29543 bench.py --gpus 4 --steps 10 --warmup 3 --split 2+2 --micro-batches 2 --no-cpu > gpurun_out/r02_bench_n4_2p2.log 2>&1
grep '^{' gpurun_out/r02_bench_n4_2p2.log | tail -1 > gpurun_out/r02_bench_n4_2p2.json; tail -c 300 gpurun_out/r02_bench_n4_2p2.log
timeout 900 $R --master-port 29544 bench_m2n.py --colocated --shape mixtral-8x22b --sizes 1,16,128,1024,3072 --iters 500 \
    > gpurun_out/r02_m2n_colo_n4.log 2>&1; grep '^{' gpurun_out/r02_m2n_colo_n4.log > gpurun_out/r02_m2n_colo_n4.jsonl; tail -c 300 gpurun_out/r02_m2n_colo_n4.log
