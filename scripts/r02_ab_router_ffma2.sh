#!/bin/bash
# exact_logits4 on FFMA2 + ALU-pipe conversions vs HEAD; router parity tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "router or route" > gpurun_out/router_tests.log 2>&1; tail -2 gpurun_out/router_tests.log
MSI_AB_BT="0,8,16" timeout 300 python scripts/ab_router_lib.py scripts/ab_libs/libmsinfer_head_router.so paper_2504_02263_b200/libmsinfer.so > gpurun_out/ab_router_ffma2.jsonl 2>&1; cat gpurun_out/ab_router_ffma2.jsonl
