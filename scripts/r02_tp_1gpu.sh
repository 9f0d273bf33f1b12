#!/bin/bash
# attention TP parity (ranks share the GPU), dense/attention tests, smoke
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attn_tp.py -q -x > gpurun_out/r02_pytest_tp.log 2>&1; tail -25 gpurun_out/r02_pytest_tp.log | cut -c1-300
timeout 600 python -m pytest tests/test_gpu_dense_gemm.py tests/test_gpu_attention.py tests/test_gpu_parity.py -q -x > gpurun_out/r02_pytest_dp.log 2>&1; tail -3 gpurun_out/r02_pytest_dp.log
