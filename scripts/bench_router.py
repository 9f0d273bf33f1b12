#!/usr/bin/env python
"""Router microbenchmark: msi_gate_topk at the bench shapes (CUDA events).
Reports time, x-read bandwidth and FMA rate (T*E*H fp32 FMAs, CUDA cores --
the bit-exact logit order rules out tensor cores)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_02263_b200 import ops  # noqa: E402

CASES = [(3072, 6144, 8, 2), (1024, 6144, 16, 4), (512, 7168, 256, 8), (4096, 7168, 256, 8), (128, 7168, 256, 8)]
for T, H, E, K in CASES:
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    wg = (torch.randn(E, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
    ws = ops.RouterWorkspace(T, E, "cuda")
    for _ in range(3):
        ops.gate_topk(x, wg, K, ws=ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    a.record()
    for _ in range(n):
        ops.gate_topk(x, wg, K, ws=ws)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / n * 1e3
    print(json.dumps({"T": T, "H": H, "E": E, "K": K, "us": us, "x_gbps": T * H * 2 / us / 1e3,
                      "tfma_per_s": T * E * H / us / 1e6}), flush=True)
