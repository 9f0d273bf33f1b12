#!/bin/bash
# PDL A/B on the M2N round trip (co-located 2->2 and 1+1, Mixtral rows), same box
set -u
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
: > gpurun_out/r02_pdl_m2n.jsonl
for rep in 1 2; do
for pdl in 0 1; do
  for mode in "--colocated" ""; do
    MSI_PDL=$pdl timeout 600 $R --master-port $((29600 + rep * 10 + pdl * 2 + ${#mode} % 2)) bench_m2n.py $mode --shape mixtral-8x22b \
      --sizes 16,1024,3072 --iters 300 --no-nccl > gpurun_out/pdl.log 2>&1
    grep '^{"metric' gpurun_out/pdl.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(json.dumps({'pdl': $pdl, 'mode': '$mode' or '1+1', 'sizes': [{k: s[k] for k in ('T','ours_p50_us','ours_graph_p50_us','ours_chain_per_trip_p50_us')} for s in d['sizes']]}))" >> gpurun_out/r02_pdl_m2n.jsonl
  done
done
done
cat gpurun_out/r02_pdl_m2n.jsonl
