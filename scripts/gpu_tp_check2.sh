#!/bin/bash
set -u
mkdir -p gpurun_out
MSI_TEST_OVERSUBSCRIBE=1 timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -k "None-2" > gpurun_out/tp_multi.log 2>&1; tail -3 gpurun_out/tp_multi.log
grep -E "^E   |Error" gpurun_out/tp_multi.log | head -20
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for TP in 2 1; do
  timeout 600 $R --master-port 2956$TP bench.py --gpus 4 --split 2+2 --tp-e $TP --micro-batches 2 --no-cpu > gpurun_out/bench_2p2_tp$TP.log 2>&1
  grep '^{' gpurun_out/bench_2p2_tp$TP.log | tail -1 > gpurun_out/bench_2p2_tp$TP.json
  python -c "
import json; d=json.load(open('gpurun_out/bench_2p2_tp$TP.json')); print('tp$TP', round(d['value']), d['config']['parallelism'], round(d['roofline']['achieved']), d['m2n']['p50_us'], d['stage_times']['T_a_ms'], d['stage_times']['T_e_ms'])" 2>&1 | tail -1
done
grep -E "Error|error" gpurun_out/bench_2p2_tp2.log | head -5
