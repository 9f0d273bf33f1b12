#!/bin/bash
# r02 2-GPU pass: default bench line (co-located 2->2), 1+1 disaggregated line,
# co-located M2N sweep vs NCCL (Mixtral rows), 1+1 M2N sweep (DBRX rows)
set -u
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02_bench_n2.log 2>&1
grep '^{' gpurun_out/r02_bench_n2.log | tail -1 > gpurun_out/r02_bench_n2.json; tail -c 300 gpurun_out/r02_bench_n2.log
timeout 600 $R --master-port 29514 bench.py --gpus 2 --steps 20 --warmup 5 --split 1+1 --micro-batches 2 > gpurun_out/r02_bench_n2_1p1.log 2>&1
grep '^{' gpurun_out/r02_bench_n2_1p1.log | tail -1 > gpurun_out/r02_bench_n2_1p1.json; tail -c 300 gpurun_out/r02_bench_n2_1p1.log
timeout 900 $R --master-port 29512 bench_m2n.py --colocated --shape mixtral-8x22b --sizes 1,16,128,1024,3072 --iters 500 \
    > gpurun_out/r02_m2n_colo_n2.log 2>&1; grep '^{' gpurun_out/r02_m2n_colo_n2.log > gpurun_out/r02_m2n_colo_n2.jsonl; tail -c 300 gpurun_out/r02_m2n_colo_n2.log
timeout 900 $R --master-port 29515 bench_m2n.py --shape mixtral-8x22b --sizes 1,16,128,1024,3072 --iters 500 \
    > gpurun_out/r02_m2n_1p1.log 2>&1; grep '^{' gpurun_out/r02_m2n_1p1.log > gpurun_out/r02_m2n_1p1.jsonl; tail -c 300 gpurun_out/r02_m2n_1p1.log
# NVLink counters of the M2N kernels on rank 0 (ncu on one rank only)
ncu --query-metrics 2>/dev/null | grep -i -E "nvl|nvlink" > gpurun_out/r02_ncu_nvl_metrics.txt
NCU_K='regex:route_dispatch|dispatch|combine' NCU_C=12 NCU_OUT=gpurun_out/r02_ncu_m2n_n2 timeout 600 \
  $R --master-port 29516 --no-python scripts/ncu_rank0.sh bench_m2n.py --colocated --shape mixtral-8x22b --sizes 3072 \
  --iters 5 --warmup 2 --no-nccl --chain 1 > gpurun_out/r02_ncu_m2n_n2.log 2>&1; tail -5 gpurun_out/r02_ncu_m2n_n2.log
