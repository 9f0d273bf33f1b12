#!/bin/bash
# N = 8 code paths on a 4-GPU box, 2 ranks per GPU (MSI_OVERSUBSCRIBE=1, gloo):
# default bench (co-located 8->8 headline + the 3+5 / 4+4 ping-pong line on
# spread slots) and the reference arm under an 8-rank launch.  Not measurements.
set -u
mkdir -p gpurun_out
export MSI_OVERSUBSCRIBE=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1"
timeout 1500 $R --master-port 29551 bench.py --gpus 8 --steps 3 --warmup 3 --no-cpu > gpurun_out/r02_n8_colo.log 2>&1; echo "colo rc=$?"
grep '^{' gpurun_out/r02_n8_colo.log | tail -1 > gpurun_out/r02_n8_colo.json
python -c "
import json; d=json.load(open('gpurun_out/r02_n8_colo.json')); print('N8', d['value'], d['parity']['routing_bit_exact']); p=d.get('pingpong'); print('PP', p and (p['value'], p['config']['workload'], p['config']['plan_source'], p['parity']))"
tail -3 gpurun_out/r02_n8_colo.log | cut -c1-300
timeout 600 $R --master-port 29552 bench.py --gpus 8 --steps 1 --warmup 1 --impl reference > gpurun_out/r02_n8_ref.log 2>&1; echo "ref rc=$?"
grep '^{' gpurun_out/r02_n8_ref.log | tail -1 | cut -c1-300
