#!/usr/bin/env python
"""One E = 256 router launch (T = 4096, DeepSeek-V3 shape) for an ncu capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_02263_b200 import ops  # noqa: E402

T, H, E, K = 4096, 7168, 256, 8
x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
wg = (torch.randn(E, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
ws = ops.RouterWorkspace(T, E, "cuda")
for _ in range(4):
    ops.gate_topk(x, wg, K, ws=ws)
torch.cuda.synchronize()
print("ok")
