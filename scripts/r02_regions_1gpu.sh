#!/bin/bash
# 1-GPU: region-path parity + dense GEMM tests, FFN A/B regions vs compact for
# n_src = 1, 2, 4, 8, and an ncu capture of the 2-sender regions GEMM1
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k regions > gpurun_out/r02_pytest_regions.log 2>&1; tail -3 gpurun_out/r02_pytest_regions.log
timeout 900 python -m pytest tests/test_gpu_dense_gemm.py tests/test_gpu_attention.py -q -x > gpurun_out/r02_pytest_dense.log 2>&1; tail -5 gpurun_out/r02_pytest_dense.log
for n in 1 2 4 8; do
  per=$((1536 / n))
  AB_NSRC=$n AB_PER=$per timeout 300 python scripts/ab_ffn_regions_1gpu.py >> gpurun_out/r02_ab_regions_1gpu.jsonl 2>gpurun_out/r02_ab_err_$n.log
done
cat gpurun_out/r02_ab_regions_1gpu.jsonl | cut -c1-250
AB_NSRC=2 AB_PER=768 AB_NCU=1 timeout 600 ncu --set full --clock-control none -k regex:grouped_gemm -c 2 \
  -o gpurun_out/r02_ncu_regions_n2 -f python scripts/ab_ffn_regions_1gpu.py > gpurun_out/r02_ncu_regions.log 2>&1; tail -3 gpurun_out/r02_ncu_regions.log
