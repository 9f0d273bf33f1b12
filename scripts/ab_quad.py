#!/usr/bin/env python
"""Quad clusters (MSI_GEMM_QUAD=1: two CTA pairs share the A operand by TMA
multicast) vs CTA pairs: expert FFN at several per-expert row counts
(including empty experts and odd 128-row tails) and the attention
projections; outputs must be bit-identical (same MMAs per tile), times are
medians of CUDA-event pairs."""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_02263_b200 import ops  # noqa: E402


def timed(fn, reps=10):
    ts = []
    for i in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def both(fn):
    res = {}
    for q in ("0", "1"):
        os.environ["MSI_GEMM_QUAD"] = q
        out = fn()
        torch.cuda.synchronize()
        res[q] = (out.clone(), timed(fn))
    os.environ["MSI_GEMM_QUAD"] = "0"
    return torch.equal(res["0"][0], res["1"][0]), res["0"][1], res["1"][1]


def main():
    H, Hp = 6144, 16384
    torch.manual_seed(0)
    shapes = [("8x768", [768 + 37 * ((e * 5) % 7 - 3) for e in range(8)]),
              ("4x1536", [1536 + 37 * ((e * 5) % 7 - 3) for e in range(4)]),
              ("8x384", [384 + 51 * ((e * 3) % 5 - 2) for e in range(8)]),
              ("ragged", [0, 1, 127, 129, 300, 0, 64, 700])]
    for name, cnt in shapes:
        E_l = len(cnt)
        rows = sum((c + 127) // 128 * 128 for c in cnt)  # 128-row aligned segments
        x = (torch.randn(rows, H, device="cuda")).to(torch.bfloat16)
        w13 = ops.pack_w13((torch.randn(E_l, Hp, H, device="cuda") / H ** 0.5).to(torch.bfloat16),
                           (torch.randn(E_l, Hp, H, device="cuda") / H ** 0.5).to(torch.bfloat16))
        w2 = (torch.randn(E_l, H, Hp, device="cuda") / Hp ** 0.5).to(torch.bfloat16)
        tot = torch.tensor(cnt, dtype=torch.int32, device="cuda")
        hb = torch.empty((rows, Hp), dtype=torch.bfloat16, device="cuda")
        same, t0, t1 = both(lambda: ops.grouped_ffn(x, tot, w13, w2, hbuf=hb))
        fl = 6.0 * sum(cnt) * H * Hp
        print(json.dumps({"ffn": name, "identical": same, "pair_ms": round(t0, 4), "quad_ms": round(t1, 4),
                          "pair_tflops": round(fl / t0 / 1e9, 1), "quad_tflops": round(fl / t1 / 1e9, 1)}), flush=True)
        del x, w13, w2, hb
    for T, N, K in ((3072, 7680, 6144), (3072, 6144, 6144), (1000, 7680, 6144), (130, 512, 1024)):
        a = torch.randn(T, K, device="cuda").to(torch.bfloat16)
        b = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
        same, t0, t1 = both(lambda: ops.dense_gemm(a, b))
        fl = 2.0 * T * N * K
        print(json.dumps({"dense": f"{T}x{N}x{K}", "identical": same, "pair_ms": round(t0, 4), "quad_ms": round(t1, 4),
                          "pair_tflops": round(fl / t0 / 1e9, 1), "quad_tflops": round(fl / t1 / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
