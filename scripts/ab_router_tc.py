#!/usr/bin/env python
"""DeepSeek-V3-shaped router (E = 256, K = 8, h = 7168): the tensor-core
candidate path (MSI_ROUTER_TC=1) vs the CUDA-core pinned-order kernels
(MSI_ROUTER_TC=0) at several T; medians of CUDA-event times, and a
bit-equality check of the two paths' outputs."""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_02263_b200 import ops  # noqa: E402


def main():
    H, E, K = 7168, 256, 8
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    wg = (torch.randn(E, H, generator=g, device="cuda") / H ** 0.5).to(torch.bfloat16)
    for T in (128, 256, 512, 1024, 2048, 4096):
        x = torch.randn(T, H, generator=g, device="cuda").to(torch.bfloat16)
        ws = ops.RouterWorkspace(T, E, "cuda")
        res = {"T": T}
        outs = {}
        for mode in ("0", "1", "1b32", "1b8"):
            os.environ["MSI_ROUTER_TC"] = mode[0]
            if mode in ("1b32", "1b8"):
                os.environ["MSI_ROUTER_TC_BT"] = mode[3:]
            else:
                os.environ.pop("MSI_ROUTER_TC_BT", None)
            ts = []
            for _ in range(15):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                o = ops.gate_topk(x, wg, K, ws)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            res[f"tc{mode}_us"] = statistics.median(ts[3:])
            outs[mode] = [t.clone() for t in o]
        res["identical"] = all(all(torch.equal(a, b) for a, b in zip(outs["0"], outs[m])) for m in outs)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
