#!/bin/bash
# M2N at 4 GPUs (gpurun --gpus 4): co-located 4->4 (Mixtral-8x22B rows) and
# disaggregated 2+2 (DBRX), per-iteration and steady-state (16 chained round
# trips) against NCCL all_to_all_single.
set -u
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29581 bench_m2n.py --colocated --shape mixtral-8x22b --sizes 1,16,128,1024,3072 \
    --iters 400 --chain 16 > gpurun_out/m2n_colo_n4.log 2>&1
grep '^{' gpurun_out/m2n_colo_n4.log > gpurun_out/m2n_colo_n4.jsonl
timeout 900 $R --master-port 29582 bench_m2n.py --shape dbrx --sizes 1,16,128,1024 --iters 400 --chain 16 \
    > gpurun_out/m2n_2p2_n4.log 2>&1
grep '^{' gpurun_out/m2n_2p2_n4.log > gpurun_out/m2n_2p2_n4.jsonl
for f in gpurun_out/m2n_colo_n4.jsonl gpurun_out/m2n_2p2_n4.jsonl; do python -c "
import json
for l in open('$f'):
    d=json.loads(l)
    if 'T' in d: print('$f'[11:], d['T'], round(d['ours_graph_p50_us'],1), round(d.get('ours_chain_per_trip_p50_us',0),1), round(d.get('nccl_graph_p50_us',0),1), round(d.get('nccl_chain_per_trip_p50_us',0),1), d['verified'], d.get('verified_chain'))
"; done
