#!/bin/bash
# router at small T: tensor-core path tiles (BT 4 / 8) vs the pinned-order path
mkdir -p gpurun_out
MSI_AB_T="64,128,256,512,1024" MSI_AB_BT="0,4,8" timeout 300 python scripts/ab_router_lib.py paper_2504_02263_b200/libmsinfer.so > gpurun_out/ab_router_smallT.jsonl 2>&1; cat gpurun_out/ab_router_smallT.jsonl
