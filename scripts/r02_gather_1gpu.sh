#!/bin/bash
# 1-GPU: region/gather parity + dense GEMM + attention tests, FFN A/B
# (region runs vs gather vs compact) for n_src = 1, 2, 4, 8
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k regions > gpurun_out/r02_pytest_regions.log 2>&1; tail -3 gpurun_out/r02_pytest_regions.log
timeout 900 python -m pytest tests/test_gpu_dense_gemm.py tests/test_gpu_attention.py -q -x > gpurun_out/r02_pytest_dense.log 2>&1; tail -5 gpurun_out/r02_pytest_dense.log
rm -f gpurun_out/r02_ab_gather_1gpu.jsonl
for n in 1 2 4 8; do
  per=$((1536 / n))
  AB_NSRC=$n AB_PER=$per timeout 300 python scripts/ab_ffn_regions_1gpu.py >> gpurun_out/r02_ab_gather_1gpu.jsonl 2>gpurun_out/r02_ab_err_$n.log
done
cut -c1-330 gpurun_out/r02_ab_gather_1gpu.jsonl
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02_bench_n1_b.json 2> gpurun_out/r02_bench_n1_b.err; tail -c 300 gpurun_out/r02_bench_n1_b.err; python -c "
import json; d=json.load(open('gpurun_out/r02_bench_n1_b.json')); print(d['value'], d['roofline']['achieved'], d['stage_times']['T_a_ms'], d['attention']['avg_launch_ms'], d['gpu_launches'])"
