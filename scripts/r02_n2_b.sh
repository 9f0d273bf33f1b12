#!/bin/bash
# 2-GPU: multi-rank parity (spread slots, co-located gather path), N=1 bench
# (refactored harness), N=2 bench with the ping-pong line
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r02_pytest_multi_b.log 2>&1; tail -3 gpurun_out/r02_pytest_multi_b.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02_bench_n1_c.json 2> gpurun_out/r02_bench_n1_c.err; tail -c 300 gpurun_out/r02_bench_n1_c.err
python -c "
import json; d=json.load(open('gpurun_out/r02_bench_n1_c.json')); print('N1', d['value'], d['roofline']['achieved'], d['stage_times']['T_a_ms'], d['gpu_launches'])"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29531 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r02_bench_n2_c.log 2>&1
grep '^{' gpurun_out/r02_bench_n2_c.log | tail -1 > gpurun_out/r02_bench_n2_c.json; tail -c 400 gpurun_out/r02_bench_n2_c.log
python -c "
import json; d=json.load(open('gpurun_out/r02_bench_n2_c.json')); print('N2', d['value'], d['roofline']['achieved'], d['stage_times']); p=d.get('pingpong'); print('PP', p and (p['value'], p['config']['workload'], p['expert_ffn'], p['stage_times']))"
