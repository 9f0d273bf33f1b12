#!/bin/bash
# ncu --set full of round-2 kernels: region gather + GEMM1 (2 senders, Mixtral-8x22B E_l=4),
# and the DS-V3 tensor-core router pieces at T=4096
set -u
mkdir -p gpurun_out
AB_NSRC=2 AB_PER=768 AB_NCU=1 AB_GATHER=1 timeout 600 ncu --set full --clock-control none -k regex:"gather_regions|grouped_gemm" -c 3 \
  -o gpurun_out/r02_ncu_gather_n2 -f python scripts/ab_ffn_regions_1gpu.py > /tmp/g.log 2>&1; tail -1 /tmp/g.log
cat > /tmp/rtc_one.py <<'PY'
import os, sys, torch
sys.path.insert(0, '.')
from paper_2504_02263_b200 import ops
os.environ["MSI_ROUTER_TC"] = "1"
H, E, K, T = 7168, 256, 8, 4096
g = torch.Generator(device="cuda"); g.manual_seed(0)
wg = (torch.randn(E, H, generator=g, device="cuda") / H ** 0.5).to(torch.bfloat16)
x = torch.randn(T, H, generator=g, device="cuda").to(torch.bfloat16)
ws = ops.RouterWorkspace(T, E, "cuda")
for _ in range(3):
    ops.gate_topk(x, wg, K, ws)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none -k regex:"wg_norm|grouped_gemm|route_kernel" -s 3 -c 3 \
  -o gpurun_out/r02_ncu_router_tc -f python /tmp/rtc_one.py > /tmp/r.log 2>&1; tail -1 /tmp/r.log
