#!/usr/bin/env python
"""Router phase timing (MSI_ROUTER_PROF=1): %globaltimer stamps of CTA 0's
phases and of the last CTA's tail, read back from the workspace (ns)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MSI_ROUTER_PROF"] = "1"
import torch  # noqa: E402

from paper_2504_02263_b200 import ops  # noqa: E402

for (T, H, E, K) in [(3072, 6144, 8, 2), (256, 6144, 8, 2), (4096, 7168, 256, 8)]:
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    wg = (torch.randn(E, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
    ws = ops.RouterWorkspace(T, E, "cuda")
    res = []
    for _ in range(6):
        ops.gate_topk(x, wg, K, ws=ws)
        torch.cuda.synchronize()
        st = ws.buf[:64].view(torch.int32).cpu().tolist()
        t = [st[i] & 0xffffffff for i in range(1, 9)]
        res.append([(v - t[0]) % (1 << 32) / 1e3 for v in t])
    names = ["entry", "after_W_stage", "after_logits", "after_topk", "ticket", "last_tail_start", "last_scan_done",
             "last_end"]
    print(json.dumps({"T": T, "E": E, "us_from_cta0_entry": dict(zip(names, [round(v, 2) for v in res[-1]]))}))
