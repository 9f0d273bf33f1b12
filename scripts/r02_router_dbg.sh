#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_dense_gemm.py -q -x -k logits 2>&1 | tail -15 | cut -c1-300
timeout 300 python - <<'PY'
import torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2504_02263_b200 import ops
H, E, K, T = 7168, 256, 8, 512
g = torch.Generator(device="cuda"); g.manual_seed(0)
wg = (torch.randn(E, H, generator=g, device="cuda") / H ** 0.5).to(torch.bfloat16)
x = torch.randn(T, H, generator=g, device="cuda").to(torch.bfloat16)
lg = ops.dense_logits(x, wg)
ref = x.float() @ wg.float().t()
print("max|tc-ref|", (lg - ref).abs().max().item(), "ref std", ref.std().item())
cb = 4 * H * 2.0 ** -24 * 1.01
xn = x.float().norm(dim=1) * 1.001
wn = wg.float().norm(dim=1) * 1.001
eps = cb * xn[:, None] * wn[None, :]
lo, hi = lg - eps, lg + eps
theta = lo.topk(K, dim=1).values[:, -1:]
cand = (hi >= theta).sum(1).float()
print("eps mean", eps.mean().item(), "candidates mean", cand.mean().item(), "max", cand.max().item())
PY
