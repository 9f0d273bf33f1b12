#!/bin/bash
set -u
mkdir -p gpurun_out
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
timeout 600 ncu --set full --import-source on --clock-control none -k regex:route_kernel -s 2 -c 1 -o gpurun_out/r02_ncu_route_tc -f python /tmp/rtc_one.py > gpurun_out/r02_ncu_route_tc.log 2>&1; tail -3 gpurun_out/r02_ncu_route_tc.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python /tmp/rtc_one.py 2>/dev/null | grep -E "route|norm|grouped" | tail -6
