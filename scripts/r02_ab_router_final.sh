#!/bin/bash
# router: final candidate pass (U=4, 2 CTAs/SM) vs the pinned-order path over T; parity tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_shapes.py -q -x -k "router or route" > gpurun_out/router_tests.log 2>&1; tail -2 gpurun_out/router_tests.log
MSI_AB_T="256,512,768,1024,2048,4096" timeout 300 python scripts/ab_router_lib.py scripts/ab_libs/libmsinfer_head_router.so paper_2504_02263_b200/libmsinfer.so > gpurun_out/ab_router_final.jsonl 2>&1; cat gpurun_out/ab_router_final.jsonl
