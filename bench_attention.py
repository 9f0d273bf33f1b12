#!/usr/bin/env python
"""Attention-stage microbenchmark: msi_decode_attention
over the paged KV cache at the workload's s (avg_seq_len 730, uniform ragged
lengths) for a sweep of batch sizes, plus the whole stage (QKV GEMM, RoPE +
append, attention, O GEMM).  Attention achieved GB/s = algorithmic bytes (K/V
rows read + q + o) / kernel time, against the measured HBM peak.

  python bench_attention.py [--shape mixtral-8x22b] [--batch 64,256,1024,3072] [--iters 20]
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
    ap.add_argument("--shape", default="mixtral-8x22b")
    ap.add_argument("--batch", default="64,256,1024,3072")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--composition", default="uniform", choices=["uniform", "fixed"])
    args = ap.parse_args()

    import torch

    from paper_2504_02263_b200 import attention as A
    from paper_2504_02263_b200 import ops
    from paper_2504_02263_b200.config import BENCH_SHAPES, WorkloadSpec

    model = BENCH_SHAPES[args.shape]
    peaks = {}
    pp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        peaks = json.load(open(pp))
    hbm = peaks.get("hbm_gbs", 6546.6)
    s = WorkloadSpec().avg_seq_len
    w = A.AttentionWeights(model, "cuda")
    for T in [int(v) for v in args.batch.split(",")]:
        st = A.AttentionStage(model, T, 1, "cuda", weights=w, avg_seq_len=s, composition=args.composition)
        c = st.cache
        x = torch.randn((T, model.hidden), device="cuda").to(torch.bfloat16)
        st.forward(x, 0)

        def run_attn():
            ops.decode_attention(st.q, c.k[0], c.v[0], c.block_table, c.lens, st.o, st.ws)

        def timed(fn):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.iters):
                fn()
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / args.iters

        # the cache (T * ~12 pages * 6 heads * 32 KB) exceeds L2 for T >= 64,
        # so back-to-back iterations read HBM
        ms_attn = timed(run_attn)
        ms_stage = timed(lambda: st.forward(x, 0))
        by = st.attn_bytes()
        rec = {"shape": args.shape, "T": T, "heads": st.n_heads, "kv_heads": st.n_kv,
               "mean_ctx": float(c.ctx_host.mean()), "kv_bytes": c.kv_bytes_read(), "attn_bytes": by,
               "splits_ws_bytes": 0 if st.ws is None else st.ws.numel(),
               "attn_ms": ms_attn, "attn_gbps": by / (ms_attn / 1e3) / 1e9, "attn_frac_hbm": by / (ms_attn / 1e3) / 1e9 / hbm,
               "stage_ms": ms_stage, "proj_tflops_in_stage": st.flops() / ((ms_stage - ms_attn) / 1e3) / 1e12
               if ms_stage > ms_attn else None}
        print(json.dumps(rec), flush=True)
        del st


if __name__ == "__main__":
    main()
