#!/usr/bin/env python
"""Expert GEMM: L2 prefetch of the weight tile k-blocks ahead (MSI_GEMM_PFB =
distance; 0 = off).  Interleaved rounds over the distances, medians of
CUDA-event times; outputs must be bit-identical to PFB = 0."""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_02263_b200 import ops  # noqa: E402

DISTS = [int(v) for v in os.environ.get("AB_PFB", "0,4,8,16,32").split(",")]


def main():
    H, Hp = 6144, 16384
    torch.manual_seed(0)
    for name, cnt in (("8x768", [768 + 37 * ((e * 5) % 7 - 3) for e in range(8)]),
                      ("4x1536", [1536 + 37 * ((e * 5) % 7 - 3) for e in range(4)])):
        E_l = len(cnt)
        rows = sum((c + 127) // 128 * 128 for c in cnt)
        x = torch.randn(rows, H, device="cuda").to(torch.bfloat16)
        w13 = ops.pack_w13((torch.randn(E_l, Hp, H, device="cuda") / H ** 0.5).to(torch.bfloat16),
                           (torch.randn(E_l, Hp, H, device="cuda") / H ** 0.5).to(torch.bfloat16))
        w2 = (torch.randn(E_l, H, Hp, device="cuda") / Hp ** 0.5).to(torch.bfloat16)
        tot = torch.tensor(cnt, dtype=torch.int32, device="cuda")
        hb = torch.empty((rows, Hp), dtype=torch.bfloat16, device="cuda")
        y = torch.zeros((rows, H), dtype=torch.bfloat16, device="cuda")
        ref = None
        same = {}
        times = {d: [] for d in DISTS}
        for r in range(8):
            for d in DISTS:
                os.environ["MSI_GEMM_PFB"] = str(d)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                ops.grouped_ffn(x, tot, w13, w2, hbuf=hb, y=y)
                b.record()
                torch.cuda.synchronize()
                if r >= 2:
                    times[d].append(a.elapsed_time(b))
                if ref is None:
                    ref = y.clone()
                same[d] = same.get(d, True) and torch.equal(y, ref)
        fl = 6.0 * sum(cnt) * H * Hp
        print(json.dumps({"ffn": name, **{f"pfb{d}_ms": round(statistics.median(times[d]), 4) for d in DISTS},
                          **{f"pfb{d}_tflops": round(fl / statistics.median(times[d]) / 1e9, 1) for d in DISTS},
                          "identical": all(same.values())}), flush=True)
        del x, w13, w2, hb, y
    os.environ["MSI_GEMM_PFB"] = "0"


if __name__ == "__main__":
    main()
