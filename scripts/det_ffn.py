#!/usr/bin/env python
"""Determinism of the expert FFN: the same call repeated (and with the L2
hints toggled) must give bit-identical valid rows."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_02263_b200 import ops, runtime  # noqa: E402
from paper_2504_02263_b200.config import as_model_spec  # noqa: E402

model = as_model_spec("mixtral-8x22b")
H, Hp = model.hidden, model.intermediate
E_l, per = 8, 768
cnt = [per + 37 * ((e * 5) % 7 - 3) for e in range(E_l)]
starts = ops.segment_starts(cnt)
rows = starts[-1] + (cnt[-1] + 127) // 128 * 128
_, w13, w2 = runtime.synth_device_weights(model, list(range(E_l)), seed=0, device="cuda")
x = torch.randn(rows, H, device="cuda").to(torch.bfloat16)
tot = torch.tensor(cnt, dtype=torch.int32, device="cuda")
outs = []
for i in range(6):
    os.environ["MSI_GEMM_L2HINT"] = str(i % 2)
    y = torch.zeros(rows, H, dtype=torch.bfloat16, device="cuda")
    ops.grouped_ffn(x, tot, w13, w2, None, y)
    torch.cuda.synchronize()
    outs.append(torch.cat([y[s:s + c] for s, c in zip(starts, cnt)]))
print("counts", cnt)
for i in range(1, 6):
    d = (outs[i].float() - outs[0].float()).abs()
    print(i, "identical" if torch.equal(outs[i], outs[0]) else f"DIFF rows={int((d.amax(1) > 0).sum())} max={d.max().item()}")
