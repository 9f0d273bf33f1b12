#!/bin/bash
# Expert-TP validation (gpurun --gpus 4): single-GPU parity suite (combine /
# dispatch / FFN regressions), every multi-GPU plan incl. the TP ones (6-rank
# plan oversubscribed), and 2+2 bench lines without / with expert TP.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_attention.py -q -x > gpurun_out/tp_parity.log 2>&1; tail -2 gpurun_out/tp_parity.log
MSI_TEST_OVERSUBSCRIBE=1 timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_pipeline.py -q -x > gpurun_out/tp_multi.log 2>&1; tail -3 gpurun_out/tp_multi.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for TP in 1 2; do
  timeout 600 $R --master-port 2956$TP bench.py --gpus 4 --split 2+2 --tp-e $TP --micro-batches 2 --no-cpu > gpurun_out/bench_2p2_tp$TP.log 2>&1
  grep '^{' gpurun_out/bench_2p2_tp$TP.log | tail -1 > gpurun_out/bench_2p2_tp$TP.json
  python -c "
import json; d=json.load(open('gpurun_out/bench_2p2_tp$TP.json')); print('tp$TP', round(d['value']), d['config']['parallelism'], round(d['roofline']['achieved']), d['m2n']['p50_us'], d['stage_times']['T_a_ms'], d['stage_times']['T_e_ms'])" 2>&1 | tail -1
done
