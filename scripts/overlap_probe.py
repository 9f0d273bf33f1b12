#!/usr/bin/env python
"""Intra-GPU overlap probe: can the HBM-bound decode attention of one
micro-batch hide under the tensor-bound expert FFN of another on the same
GPU?  Times attention alone, the grouped FFN alone at several persistent grid
sizes (MSI_GEMM_GRID), and both launched concurrently on two streams (FFN
first, so its CTAs hold their SMs and attention takes the rest)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_02263_b200 import attention as A, ops  # noqa: E402
from paper_2504_02263_b200.config import as_model_spec  # noqa: E402

T = int(os.environ.get("PROBE_T", "1536"))
model = as_model_spec("mixtral-8x22b")
dev = torch.device("cuda:0")
st = A.AttentionStage(model, T, 1, dev, avg_seq_len=730, seed=1)
x = torch.randn(T, model.hidden, device=dev).to(torch.bfloat16)
E, H, Hp = 8, model.hidden, model.intermediate
te = T * 2 // E
g = torch.Generator().manual_seed(te)
totals = [max(1, int(te * (0.95 + 0.1 * torch.rand(1, generator=g).item()))) for _ in range(E)]
rows = sum((t + 127) // 128 * 128 for t in totals)
xr = torch.randn(rows, H, device=dev).to(torch.bfloat16)
tot = torch.tensor(totals, dtype=torch.int32, device=dev)
w13 = (torch.randn(E, 2 * Hp, H, device=dev) / H ** 0.5).to(torch.bfloat16)
w2 = (torch.randn(E, H, Hp, device=dev) / Hp ** 0.5).to(torch.bfloat16)
hbuf = torch.empty(rows, Hp, dtype=torch.bfloat16, device=dev)
y = torch.empty(rows, H, dtype=torch.bfloat16, device=dev)
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fa=None, fb=None, reps=7):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if fa:
            sa.wait_event(e0)
            with torch.cuda.stream(sa):
                fa()
                ea.record(sa)
        if fb:
            sb.wait_event(e0)
            with torch.cuda.stream(sb):
                fb()
                eb.record(sb)
        torch.cuda.synchronize()
        t = [e0.elapsed_time(e) for e, f in ((ea, fa), (eb, fb)) if f]
        out.append(max(t))
    return statistics.median(out[1:])


attn = lambda: st.forward(x, 0)  # noqa: E731
ffn = lambda: ops.grouped_ffn(xr, tot, w13, w2, hbuf, y)  # noqa: E731
res = {"T": T, "t_e": te, "attn_ms": timed(fb=attn)}
for grid in (148, 136, 128, 120, 112, 96):
    os.environ["MSI_GEMM_GRID"] = str(grid)
    f = timed(fa=ffn)
    both = timed(fa=ffn, fb=attn)
    res[f"grid{grid}"] = {"ffn_ms": round(f, 3), "both_ms": round(both, 3),
                          "sum_ms": round(f + res["attn_ms"], 3), "gain": round((f + res["attn_ms"]) / both, 3)}
os.environ.pop("MSI_GEMM_GRID", None)
print(json.dumps(res), flush=True)
