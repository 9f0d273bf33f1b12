#!/bin/bash
# router TC candidate pass: HEAD (one warp per token) vs balanced items; BT sweep
mkdir -p gpurun_out
MSI_AB_BT="0,8,12,16" timeout 300 python scripts/ab_router_lib.py scripts/ab_libs/libmsinfer_head_router.so paper_2504_02263_b200/libmsinfer.so > gpurun_out/ab_router_balance.jsonl 2>&1; tail -5 gpurun_out/ab_router_balance.jsonl
