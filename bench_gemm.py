#!/usr/bin/env python
"""Expert grouped-GEMM microbenchmark (msi_grouped_ffn: GEMM1 gate/up+SiLU and
GEMM2 down) on a Mixtral-8x22B-shaped expert group, for a sweep of tokens per
expert t_e.  Reports algorithmic TFLOP/s (6 * rows * h * h') against the
measured bf16 peaks.  MSI_GEMM_CG=1|2 selects the CTA-group variant.

  python bench_gemm.py [--experts 8] [--te 256,768,1536] [--iters 10]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--hidden", type=int, default=6144)
    ap.add_argument("--inter", type=int, default=16384)
    ap.add_argument("--te", default="64,256,768,1536")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--exact", action="store_true", help="every expert gets exactly t_e rows (no raggedness)")
    ap.add_argument("--ab", type=int, default=0,
                    help="interleaved A/B of the 1-CTA and CTA-pair kernels: N alternating rounds, medians")
    ap.add_argument("--ab-env", default="",
                    help="A/B an env setting instead, e.g. MSI_GEMM_PREFETCH=0:8 (variant 1 : variant 2)")
    args = ap.parse_args()

    import torch

    from paper_2504_02263_b200 import ops

    torch.manual_seed(0)
    E, H, Hp = args.experts, args.hidden, args.inter
    dev = torch.device("cuda:0")
    w13 = (torch.randn(E, 2 * Hp, H, device=dev) / H ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn(E, H, Hp, device=dev) / Hp ** 0.5).to(torch.bfloat16)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    out = []
    for te in [int(v) for v in args.te.split(",")]:
        # realistic ragged loads: +-5% around te
        g = torch.Generator().manual_seed(te)
        totals = [te if args.exact else max(1, int(te * (0.95 + 0.1 * torch.rand(1, generator=g).item())))
                  for _ in range(E)]
        rows = sum((t + 127) // 128 * 128 for t in totals)
        x = torch.randn(rows, H, device=dev).to(torch.bfloat16)
        tot = torch.tensor(totals, dtype=torch.int32, device=dev)
        hbuf = torch.empty(rows, Hp, dtype=torch.bfloat16, device=dev)
        y = torch.empty(rows, H, dtype=torch.bfloat16, device=dev)
        if args.ab:
            from paper_2504_02263_b200 import _lib
            lib = _lib.load()
            per = {1: [], 2: []}
            env_key, env_vals = (args.ab_env.split("=")[0], args.ab_env.split("=")[1].split(":")) if args.ab_env else (None, None)
            for rnd in range(args.ab):
                for cg in ((1, 2) if rnd % 2 == 0 else (2, 1)):
                    if env_key:
                        os.environ[env_key] = env_vals[cg - 1]
                    else:
                        lib.msi_set_gemm_cta_group(cg)
                    for _ in range(2):
                        ops.grouped_ffn(x, tot, w13, w2, hbuf, y)
                    torch.cuda.synchronize()
                    s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s0.record()
                    for _ in range(args.iters):
                        ops.grouped_ffn(x, tot, w13, w2, hbuf, y)
                    e0.record()
                    torch.cuda.synchronize()
                    per[cg].append(s0.elapsed_time(e0) / args.iters)
            lib.msi_set_gemm_cta_group(0)
            flops = 6.0 * sum(totals) * H * Hp
            rec = {"ab": args.ab, "ab_env": args.ab_env or "cta_group 1:2", "te": te, "exact": args.exact, "rows": sum(totals),
                   "odd_tiles": sum(((t + 127) // 128) % 2 for t in totals)}
            for cg in (1, 2):
                ms = sorted(per[cg])[len(per[cg]) // 2]
                rec[f"cg{cg}_ms"] = ms
                rec[f"cg{cg}_tflops"] = flops / (ms / 1e3) / 1e12
            rec["cg2_over_cg1"] = rec["cg1_ms"] / rec["cg2_ms"]
            out.append(rec)
            print(json.dumps(rec), flush=True)
            continue
        for _ in range(3):
            ops.grouped_ffn(x, tot, w13, w2, hbuf, y)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.iters):
            ops.grouped_ffn(x, tot, w13, w2, hbuf, y)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / args.iters
        flops = 6.0 * sum(totals) * H * Hp
        tf = flops / (ms / 1e3) / 1e12
        rec = {"cg": os.environ.get("MSI_GEMM_CG", "default"), "te": te, "exact": args.exact, "rows": sum(totals), "ms": ms,
               "tflops": tf, "frac_burst": tf / peaks.get("bf16_tflops", 1677.4),
               "frac_sustained": tf / peaks.get("bf16_tflops_sustained", 1404.8),
               "weight_gbps": E * 3 * H * Hp * 2 / (ms / 1e3) / 1e9}
        out.append(rec)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
