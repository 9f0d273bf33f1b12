#!/bin/bash
# candidate pass: loads in flight (MSI_EXACT_U) x register budget (MSI_ROUTE_LB)
mkdir -p gpurun_out
MSI_AB_BT="0,8" timeout 300 python scripts/ab_router_lib.py scripts/ab_libs/libmsinfer_head_router.so scripts/ab_libs/libmsinfer_u2lb3.so scripts/ab_libs/libmsinfer_u2lb2.so scripts/ab_libs/libmsinfer_u3lb2.so scripts/ab_libs/libmsinfer_u4lb2.so > gpurun_out/ab_router_u.jsonl 2>&1; cat gpurun_out/ab_router_u.jsonl
