#!/bin/bash
# 2-GPU pass: edge-case parity tests, co-located M2N sweep vs NCCL (Mixtral-8x22B
# rows, the bench's default layout), and the default bench line at N = 2.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "nonfinite or concentrated or empty" > gpurun_out/edge.log 2>&1; tail -2 gpurun_out/edge.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
    bench_m2n.py --colocated --shape mixtral-8x22b --sizes 1,16,128,512,1024,3072 --iters ${ITERS:-500} \
    > gpurun_out/m2n_colo_n2.log 2>&1; grep '^{' gpurun_out/m2n_colo_n2.log > gpurun_out/m2n_colo_n2.jsonl; tail -c 600 gpurun_out/m2n_colo_n2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2.log 2>&1
grep '^{' gpurun_out/bench_n2.log | tail -1 > gpurun_out/bench_n2.json; tail -c 700 gpurun_out/bench_n2.log
