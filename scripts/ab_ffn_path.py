#!/usr/bin/env python
"""msi_expert_ffn (through the M2N receive buffer) vs msi_grouped_ffn on the
same rows packed compactly, on the bench's N = 1 shape, interleaved, medians.
Uses only router / dispatch / expert_wait / expert_ffn / combine, so it runs
against older builds too (PYTHONPATH=<tree> python scripts/ab_ffn_path.py)."""
import json
import os
import statistics
import sys

import torch

from paper_2504_02263_b200 import ops, runtime
from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec


def ev():
    return torch.cuda.Event(enable_timing=True)


model = as_model_spec("mixtral-8x22b")
T = 3072
g = runtime.M2NGroup(model, DeploymentPlan(n_a=1, n_e=1, m=1, b_a=T, colocated=True), rank=0)
wg, w13, w2 = runtime.synth_device_weights(model, runtime.local_experts(g), seed=0, device=g.device)
layer = runtime.MoEDecodeLayer(g, wg=wg, w13=w13, w2=w2)
torch.manual_seed(0)
x = torch.randn(T, model.hidden, device=g.device).to(torch.bfloat16)
r = layer.router(x, 0)
cnt = r.cnt.cpu().tolist()
starts = ops.segment_starts(cnt)
rows = starts[-1] + (cnt[-1] + 127) // 128 * 128
xc = torch.randn(rows, model.hidden, device=g.device).to(torch.bfloat16)
tot = torch.tensor(cnt, dtype=torch.int32, device=g.device)
hbuf = torch.empty(rows, model.intermediate, dtype=torch.bfloat16, device=g.device)
y = torch.empty(rows, model.hidden, dtype=torch.bfloat16, device=g.device)
res = {"expert_ffn_ms": [], "grouped_ffn_ms": []}
for i in range(14):
    r = layer.router(x, 0)
    layer.dispatch(x, r, 0)
    layer.expert_wait(0)
    s, e = ev(), ev()
    s.record()
    layer.expert_ffn(0)
    e.record()
    layer.combine(r)
    c0, c1 = ev(), ev()
    c0.record()
    ops.grouped_ffn(xc, tot, w13, w2, hbuf, y)
    c1.record()
    torch.cuda.synchronize()
    res["expert_ffn_ms"].append(s.elapsed_time(e))
    res["grouped_ffn_ms"].append(c0.elapsed_time(c1))
out = {k: statistics.median(v[2:]) for k, v in res.items()}
out["tree"] = os.path.dirname(os.path.dirname(os.path.abspath(runtime.__file__)))
print(json.dumps(out))
