#!/usr/bin/env python
"""One-GPU A/B of the expert FFN with n_src senders' receive regions
(msi_grouped_ffn_regions, GEMM1 loading A as region runs) against the same
rows packed compactly per expert (msi_grouped_ffn): Mixtral-8x22B, E_l local
experts, counts ~ T*K/E per (expert, sender) with ragged noise.  Prints
medians; AB_NCU=1 runs the regions variant only (for ncu)."""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_02263_b200 import ops, runtime  # noqa: E402
from paper_2504_02263_b200.config import as_model_spec  # noqa: E402


def main():
    model = as_model_spec(os.environ.get("AB_SHAPE", "mixtral-8x22b"))
    n_src = int(os.environ.get("AB_NSRC", "2"))
    E_l = int(os.environ.get("AB_EL", "4"))
    per = int(os.environ.get("AB_PER", "768"))  # mean rows per (expert, sender)
    cap = int(os.environ.get("AB_CAP", str(per * 2)))
    rng = np.random.default_rng(0)
    counts = np.clip(rng.normal(per, per * 0.06, size=(n_src, E_l)).round(), 0, cap).astype(np.int64)
    torch.cuda.set_device(0)
    _, w13, w2 = runtime.synth_device_weights(model, list(range(E_l)), seed=0, device="cuda")
    H = model.hidden
    x_reg = torch.randn((E_l * n_src * cap, H), device="cuda").to(torch.bfloat16)
    tot = counts.sum(0)
    starts = ops.segment_starts(tot.tolist())
    rows = starts[-1] + (int(tot[-1]) + 127) // 128 * 128
    xc = torch.zeros((rows, H), dtype=torch.bfloat16, device="cuda")
    for e in range(E_l):
        o = starts[e]
        for s in range(n_src):
            b = (e * n_src + s) * cap
            xc[o:o + counts[s, e]] = x_reg[b:b + counts[s, e]]
            o += counts[s, e]
    tt = torch.tensor(tot, dtype=torch.int32, device="cuda")
    hc = torch.empty((rows, model.intermediate), dtype=torch.bfloat16, device="cuda")
    yc = torch.empty((rows, H), dtype=torch.bfloat16, device="cuda")
    y_reg = torch.zeros_like(x_reg)
    hb = torch.empty((rows + 128, model.intermediate), dtype=torch.bfloat16, device="cuda")
    flops = 6.0 * tot.sum() * H * model.intermediate
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    if os.environ.get("AB_NCU") == "1":
        for _ in range(3):
            ops.grouped_ffn_regions(x_reg, counts, cap, w13, w2, y_reg, hb,
                                    gather=os.environ.get("AB_GATHER") == "1")
        torch.cuda.synchronize()
        return
    res = {"regions_ms": [], "compact_ms": [], "gather_ms": []}
    y_g = torch.zeros_like(x_reg)
    for _ in range(int(os.environ.get("AB_ITERS", "12"))):
        a, b = ev(), ev()
        a.record()
        ops.grouped_ffn_regions(x_reg, counts, cap, w13, w2, y_reg, hb)
        b.record()
        c, d = ev(), ev()
        c.record()
        ops.grouped_ffn(xc, tt, w13, w2, hc, yc)
        d.record()
        g0, g1 = ev(), ev()
        g0.record()
        ops.grouped_ffn_regions(x_reg, counts, cap, w13, w2, y_g, hb, gather=True)
        g1.record()
        torch.cuda.synchronize()
        res["gather_ms"].append(g0.elapsed_time(g1))
        res["regions_ms"].append(a.elapsed_time(b))
        res["compact_ms"].append(c.elapsed_time(d))
    # bit-exact: the same rows through the two layouts
    same = True
    for e in range(E_l):
        o = starts[e]
        for s in range(n_src):
            bb = (e * n_src + s) * cap
            same &= torch.equal(y_reg[bb:bb + counts[s, e]], yc[o:o + counts[s, e]])
            same &= torch.equal(y_g[bb:bb + counts[s, e]], yc[o:o + counts[s, e]])
            o += counts[s, e]
    out = {k: statistics.median(v[2:]) for k, v in res.items()}
    out["regions_tflops"] = flops / (out["regions_ms"] * 1e-3) / 1e12
    out["compact_tflops"] = flops / (out["compact_ms"] * 1e-3) / 1e12
    out["gather_tflops"] = flops / (out["gather_ms"] * 1e-3) / 1e12
    out.update(n_src=n_src, E_l=E_l, per=per, bit_exact=bool(same), counts=counts.tolist(),
               cg=os.environ.get("MSI_GEMM_CG", "2"))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
