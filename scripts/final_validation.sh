#!/bin/bash
# End-of-round validation on a 4-GPU box: the full GPU suite (8-rank plans
# oversubscribed 2 per GPU), smoke, and the default bench lines at N = 1, 2, 4.
set -u
mkdir -p gpurun_out
MSI_TEST_OVERSUBSCRIBE=1 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; tail -2 gpurun_out/final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench_n1.log 2>&1; grep '^{' gpurun_out/final_bench_n1.log | tail -1 > gpurun_out/final_bench_n1.json
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N \
      bench.py --gpus $N > gpurun_out/final_bench_n$N.log 2>&1
  grep '^{' gpurun_out/final_bench_n$N.log | tail -1 > gpurun_out/final_bench_n$N.json
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref_n1.log 2>&1; grep '^{' gpurun_out/final_ref_n1.log | tail -1 > gpurun_out/final_ref_n1.json
for f in gpurun_out/final_bench_n*.json gpurun_out/final_ref_n1.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['n_gpus'], round(d['value']), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('m2n') or {}).get('p50_us'), (d.get('clocks') or {}).get('sm_mhz'))"; done
