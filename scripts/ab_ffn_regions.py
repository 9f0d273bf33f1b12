#!/usr/bin/env python
"""Same-box A/B of the expert FFN on the bench's N = 1 shape (Mixtral-8x22B,
T = 3072 routed tokens, 8 local experts): msi_expert_ffn reading A as runs of
the receive regions vs msi_grouped_ffn on the same rows packed compactly
(one 128-row box per tile).  Interleaved rounds, medians (ms and TFLOP/s).
Also times the fused router + dispatch against router + dispatch."""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_02263_b200 import ops, runtime  # noqa: E402
from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    model = as_model_spec(os.environ.get("AB_SHAPE", "mixtral-8x22b"))
    T = int(os.environ.get("AB_T", "3072"))
    g = runtime.M2NGroup(model, DeploymentPlan(n_a=1, n_e=1, m=1, b_a=T, colocated=True), rank=0)
    wg, w13, w2 = runtime.synth_device_weights(model, runtime.local_experts(g), seed=0, device=g.device)
    layer = runtime.MoEDecodeLayer(g, wg=wg, w13=w13, w2=w2)
    x = torch.randn(T, model.hidden, device=g.device).to(torch.bfloat16)
    r = layer.route_dispatch(x, 0)
    layer.expert_step(0)
    layer.combine(r)
    torch.cuda.synchronize()
    cnt = r.cnt.cpu().tolist()
    starts = ops.segment_starts(cnt)
    rows = starts[-1] + (cnt[-1] + 127) // 128 * 128
    recv = g.recv_view(0)
    xc = torch.zeros(rows, model.hidden, dtype=torch.bfloat16, device=g.device)
    for e, (s0, c) in enumerate(zip(starts, cnt)):
        xc[s0:s0 + c] = recv[e * T: e * T + c]
    tot = torch.tensor(cnt, dtype=torch.int32, device=g.device)
    hbuf = torch.empty(rows, model.intermediate, dtype=torch.bfloat16, device=g.device)
    y = torch.empty(rows, model.hidden, dtype=torch.bfloat16, device=g.device)
    flops = 6.0 * T * model.topk * model.hidden * model.intermediate
    res = {"regions_ms": [], "compact_ms": [], "route_dispatch_us": [], "router_plus_dispatch_us": []}
    for _ in range(int(os.environ.get("AB_ITERS", "12"))):
        a0, a1, b0, b1 = ev(), ev(), ev(), ev()
        a0.record()
        r = layer.route_dispatch(x, 0)
        a1.record()
        layer.expert_wait(0)
        s, e = ev(), ev()
        s.record()
        layer.expert_ffn(0)
        e.record()
        layer.combine(r)
        b0.record()
        r = layer.router(x, 0)
        layer.dispatch(x, r, 0)
        b1.record()
        layer.expert_step(0)
        layer.combine(r)
        c0, c1 = ev(), ev()
        c0.record()
        ops.grouped_ffn(xc, tot, w13, w2, hbuf, y)
        c1.record()
        torch.cuda.synchronize()
        res["regions_ms"].append(s.elapsed_time(e))
        res["compact_ms"].append(c0.elapsed_time(c1))
        res["route_dispatch_us"].append(a0.elapsed_time(a1) * 1e3)
        res["router_plus_dispatch_us"].append(b0.elapsed_time(b1) * 1e3)
    # fused router + dispatch under other CTA tiles (MSI_ROUTER_TILE=TTxTExBT)
    for tile in ("1x8x8", "2x8x16", "4x8x32"):
        os.environ["MSI_ROUTER_TILE"] = tile
        ts = []
        for _ in range(10):
            a0, a1 = ev(), ev()
            a0.record()
            r = layer.route_dispatch(x, 0)
            a1.record()
            layer.expert_step(0)
            layer.combine(r)
            torch.cuda.synchronize()
            ts.append(a0.elapsed_time(a1) * 1e3)
        res[f"route_dispatch_us_{tile}"] = ts
        del os.environ["MSI_ROUTER_TILE"]
    assert g.status() == 0
    out = {k: statistics.median(v[2:] if len(v) > 2 else v) for k, v in res.items()}
    out["regions_tflops"] = flops / (out["regions_ms"] * 1e-3) / 1e12
    out["compact_tflops"] = flops / (out["compact_ms"] * 1e-3) / 1e12
    out.update(shape=model.name, T=T, counts=cnt)
    print(json.dumps(out))
    g.close()


if __name__ == "__main__":
    main()
