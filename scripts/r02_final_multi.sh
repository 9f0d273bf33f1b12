#!/bin/bash
# final code: default bench lines at N = 2 and N = 4 (co-located headline + ping-pong line)
set -u
mkdir -p gpurun_out
for n in 2 4; do
  timeout 1200 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800 + n)) bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r02_bench_final_n$n.log 2>&1
  echo "N=$n rc=$?"
  grep '^{' gpurun_out/r02_bench_final_n$n.log | tail -1 > gpurun_out/r02_bench_final_n$n.json
  python -c "
import json; d=json.load(open('gpurun_out/r02_bench_final_n$n.json')); m=d['m2n']; p=d.get('pingpong') or {}
print('N=$n', int(d['value']), int(d['value_per_gpu']), round(d['roofline']['achieved']), 'm2n', round(m['p50_us'],1), round(m['roofline']['frac_nominal'],3), round(m['steady_state']['roofline']['frac_nominal'],3), 'pp', int(p.get('value') or 0), p.get('config',{}).get('workload'), d['parity']['routing_bit_exact'], d['clocks']['sm_mhz'])"
done
