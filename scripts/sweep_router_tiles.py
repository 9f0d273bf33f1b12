#!/usr/bin/env python
"""Router tile-shape sweep (MSI_ROUTER_TILE=TTxTExBT overrides): time per shape
and check the outputs are bit-identical to the default choice."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_02263_b200 import ops  # noqa: E402

CASES = {(3072, 6144, 8, 2): ["4x8x32", "2x8x16", "1x8x8", "4x8x16", "2x8x8", "8x4x32", "4x4x16"],
         (1024, 6144, 16, 4): ["4x16x32", "2x16x16", "1x16x8", "4x8x16", "2x8x8", "1x8x8"],
         (4096, 7168, 256, 8): ["4x16x16", "4x16x4", "8x8x32"],
         (512, 7168, 256, 8): ["4x16x4", "2x16x4"]}
if sys.argv[1:] == ["e256"]:  # E = 256 only (re-sweep after the FFMA2 logits loop)
    CASES = {(4096, 7168, 256, 8): ["4x16x28", "8x8x32", "8x8x24", "8x4x32", "4x8x28", "2x16x28"],
             (2048, 7168, 256, 8): ["4x16x16", "8x8x16", "4x8x16", "2x16x16"],
             (512, 7168, 256, 8): ["4x16x4", "2x16x4", "4x8x4", "8x8x8"]}
for (T, H, E, K), tiles in CASES.items():
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    wg = (torch.randn(E, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
    ws = ops.RouterWorkspace(T, E, "cuda")
    os.environ.pop("MSI_ROUTER_TILE", None)
    ref = [t.clone() for t in ops.gate_topk(x, wg, K, ws=ws)]
    for tile in ["default"] + tiles:
        if tile == "default":
            os.environ.pop("MSI_ROUTER_TILE", None)
        else:
            os.environ["MSI_ROUTER_TILE"] = tile
        out = ops.gate_topk(x, wg, K, ws=ws)
        torch.cuda.synchronize()
        same = all(torch.equal(a, b) for a, b in zip(out, ref))
        for _ in range(3):
            ops.gate_topk(x, wg, K, ws=ws)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            ops.gate_topk(x, wg, K, ws=ws)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 20 * 1e3
        print(json.dumps({"T": T, "E": E, "tile": tile, "us": round(us, 1), "same": same}), flush=True)
