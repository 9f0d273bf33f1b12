#!/usr/bin/env python
"""Fused router + dispatch (msi_route_dispatch) at the N = 1 bench shape
(Mixtral-8x22B, T = 3072, co-located) under router tiles MSI_ROUTER_TILE."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_02263_b200 import runtime
from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec

model = as_model_spec("mixtral-8x22b")
T = int(os.environ.get("AB_T", "3072"))
g = runtime.M2NGroup(model, DeploymentPlan(n_a=1, n_e=1, m=1, b_a=T, colocated=True), rank=0)
wg, w13, w2 = runtime.synth_device_weights(model, runtime.local_experts(g), seed=0, device=g.device)
layer = runtime.MoEDecodeLayer(g, wg=wg, w13=w13, w2=w2)
x = torch.randn(T, model.hidden, device=g.device).to(torch.bfloat16)
res = {}
for tile in ("default", "4x8x24", "4x8x16", "2x8x16", "2x8x8", "1x8x8", "1x8x4", "4x8x32", "2x8x32", "8x8x32"):
    if tile == "default":
        os.environ.pop("MSI_ROUTER_TILE", None)
    else:
        os.environ["MSI_ROUTER_TILE"] = tile
    ts = []
    for i in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = layer.route_dispatch(x, 0)
        b.record()
        layer.expert_step(0)
        layer.combine(r)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b) * 1e3)
    res[tile] = round(statistics.median(ts), 1)
assert g.status() == 0
print(json.dumps({"T": T, "route_dispatch_us": res}))
