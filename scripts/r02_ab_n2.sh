#!/bin/bash
# 2-GPU same-box A/B: expert FFN on receive-region runs vs compact rows; then the
# new dense-GEMM tests (1 GPU of the pair)
set -u
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29521 scripts/ab_ffn_regions_n2.py > gpurun_out/r02_ab_regions_n2.log 2>&1; grep '^{' gpurun_out/r02_ab_regions_n2.log; tail -3 gpurun_out/r02_ab_regions_n2.log
MSI_GEMM_CG=1 timeout 600 $R --master-port 29522 scripts/ab_ffn_regions_n2.py > gpurun_out/r02_ab_regions_n2_cg1.log 2>&1; grep '^{' gpurun_out/r02_ab_regions_n2_cg1.log
timeout 900 python -m pytest tests/test_gpu_dense_gemm.py tests/test_gpu_attention.py -q -x > gpurun_out/r02_pytest_dense.log 2>&1; tail -15 gpurun_out/r02_pytest_dense.log
