#!/bin/bash
# Multi-GPU validation pass (gpurun --gpus 4): new parity edge cases, the
# multi-GPU parity suite with 8-rank plans oversubscribed onto 4 GPUs, and
# the default bench layout at N = 2, 4 (planner -> co-located).
set -u
mkdir -p gpurun_out
nvidia-smi -L
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "nonfinite or concentrated or empty" > gpurun_out/edge.log 2>&1; tail -3 gpurun_out/edge.log
MSI_TEST_OVERSUBSCRIBE=1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi_oversub.log 2>&1; tail -3 gpurun_out/multi_oversub.log
for N in ${NS:-2 4}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/bench_n$N.log 2>&1
  grep '^{' gpurun_out/bench_n$N.log | tail -1 > gpurun_out/bench_n$N.json; tail -c 400 gpurun_out/bench_n$N.log
done
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench_n1_m2n.log 2>&1
grep '^{' gpurun_out/bench_n1_m2n.log > gpurun_out/bench_n1_m2n.json
