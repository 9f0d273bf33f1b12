#!/bin/bash
cat > /tmp/rd1.py <<'PY'
import os, sys, torch
sys.path.insert(0, '.')
from paper_2504_02263_b200 import runtime
from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec
m = as_model_spec("mixtral-8x22b"); T = 3072
g = runtime.M2NGroup(m, DeploymentPlan(n_a=1, n_e=1, m=1, b_a=T, colocated=True), rank=0)
wg, w13, w2 = runtime.synth_device_weights(m, runtime.local_experts(g), seed=0, device=g.device)
layer = runtime.MoEDecodeLayer(g, wg=wg, w13=w13, w2=w2)
x = torch.randn(T, m.hidden, device=g.device).to(torch.bfloat16)
for _ in range(3):
    r = layer.route_dispatch(x, 0); layer.expert_step(0); layer.combine(r)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gate_topk -s 2 -c 1 -o gpurun_out/r02_ncu_route_n1 -f python /tmp/rd1.py > /tmp/n.log 2>&1; tail -2 /tmp/n.log
