#!/usr/bin/env python
"""Calibrate the SPEC cost models from B200 measurements.

Times the two compute stages of the decode step with CUDA events on one GPU
and writes the reference's profile CSV:

* ``expert,b_e,seconds``   -- msi_grouped_ffn (GEMM1 gate/up+SiLU, GEMM2 down)
  over E_l local experts holding t_e tokens each (b_e = E_l * t_e rows);
* ``attention,b_a,seconds`` -- the attention stage at the workload's s
  (the KV stand-in, reading b_a * s * 2 * (h/g) * 2 bytes);
* ``nvlink-peer,message_bytes,utilization`` -- from a ``bench_m2n.py`` JSONL
  (``--m2n``): one-way dispatch bytes per pair / p50 time / 900 GB/s.

Then fits k1..k4 with ``perf_model.calibrate`` (held-out check: fit on every
other point, predict the rest) and, given a bench.py JSON line (``--bench``),
compares the measured step with Eq. 5 evaluated from the fitted model.

  python calibrate.py --shape mixtral-8x22b --experts-local 8 \
      --out profiles/r01_profile_8x22b.csv [--m2n profiles/r01_m2n_n2.jsonl] [--bench b.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2504_02263_b200 import perf_model as PM  # noqa: E402
from paper_2504_02263_b200.config import BENCH_SHAPES, WorkloadSpec  # noqa: E402

NVLINK_BPS = 900e9


def time_ms(fn, iters: int) -> float:
    import torch
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def profile_expert(model, e_l: int, tes: list, iters: int) -> list:
    import torch
    from paper_2504_02263_b200 import ops
    dev = torch.device("cuda:0")
    H, Hp = model.hidden, model.intermediate
    g = torch.Generator(device=dev).manual_seed(0)
    w13 = (torch.randn(e_l, 2 * Hp, H, device=dev, generator=g) / H ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn(e_l, H, Hp, device=dev, generator=g) / Hp ** 0.5).to(torch.bfloat16)
    rows_out = []
    for te in tes:
        rows = e_l * ((te + 127) // 128 * 128)
        x = torch.randn(rows, H, device=dev, generator=g).to(torch.bfloat16)
        tot = torch.full((e_l,), te, dtype=torch.int32, device=dev)
        hbuf = torch.empty(rows, Hp, dtype=torch.bfloat16, device=dev)
        y = torch.empty(rows, H, dtype=torch.bfloat16, device=dev)
        ms = time_ms(lambda: ops.grouped_ffn(x, tot, w13, w2, hbuf, y), iters)
        rows_out.append(("expert", e_l * te, ms / 1e3))
        del x, hbuf, y
    return rows_out


def profile_attention(model, seq_len: int, bas: list, iters: int) -> list:
    """T_a(b_a): the real attention stage (QKV projection, RoPE + KV append,
    paged decode attention at mean context seq_len, output projection)."""
    from paper_2504_02263_b200 import attention as A
    dev = torch_device()
    w = A.AttentionWeights(model, dev, seed=0)
    out = []
    for b in bas:
        st = A.AttentionStage(model, b, 1, dev, weights=w, avg_seq_len=seq_len, seed=b)
        x = st.y.clone().normal_()
        ms = time_ms(lambda: st.forward(x, 0), iters)
        out.append(("attention", b, ms / 1e3))
        del st, x
    return out


def torch_device():
    import torch
    return torch.device("cuda:0")


def util_from_m2n(path: str) -> list:
    out = []
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        r = json.loads(line)
        if "dispatch_only_p50_us" not in r or "pair_bytes_avg" not in r:
            continue
        gbps = r["ingress_bytes_busiest"] / (r["dispatch_only_p50_us"] * 1e-6)
        out.append(("nvlink-peer", int(r["pair_bytes_avg"]), min(gbps / NVLINK_BPS, 1.0)))
    return out


def held_out(points: list, kind: str) -> dict:
    pts = sorted((b, t) for _, b, t in points)
    fit_pts, test_pts = pts[::2], pts[1::2]
    if len({b for b, _ in fit_pts}) < 2 or not test_pts:
        return {}
    f = PM.calibrate(fit_pts, kind)
    errs = [abs(f(b) - t) / t for b, t in test_pts]
    return {"fit_on": [b for b, _ in fit_pts], "held_out": [b for b, _ in test_pts],
            "max_rel_err": max(errs)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="mixtral-8x22b", choices=sorted(BENCH_SHAPES))
    ap.add_argument("--experts-local", type=int, default=None, help="E_l (default: all experts)")
    ap.add_argument("--te", default="128,256,384,512,768,1024,1536,2048")
    ap.add_argument("--ba", default="256,512,1024,1536,2048,3072")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--m2n", default=None, help="bench_m2n.py JSONL for the UtilCurve table")
    ap.add_argument("--bench", default=None, help="bench.py JSON line to check against Eq. 5")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    model = BENCH_SHAPES[args.shape]
    e_l = args.experts_local or model.experts
    s = WorkloadSpec().avg_seq_len
    exp_rows = profile_expert(model, e_l, [int(v) for v in args.te.split(",")], args.iters)
    att_rows = profile_attention(model, s, [int(v) for v in args.ba.split(",")], args.iters)
    util_rows = util_from_m2n(args.m2n) if args.m2n else []
    out = args.out or os.path.join(ROOT, "gpurun_out", f"profile_{args.shape}.csv")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    PM.write_profile(out, exp_rows + att_rows, util_rows)
    cm = PM.cost_model_from_profile(out)
    rep = {"shape": args.shape, "experts_local": e_l, "seq_len": s, "profile": os.path.relpath(out, ROOT),
           "k1_s_per_tok": cm.k1, "k2_s": cm.k2, "k3_s_per_tok": cm.k3, "k4_s": cm.k4,
           "expert_fit_residual_rms_s": PM.calibrate([r[1:] for r in exp_rows], "expert").residual_rms,
           "attention_fit_residual_rms_s": PM.calibrate([r[1:] for r in att_rows], "attention").residual_rms,
           "expert_held_out": held_out(exp_rows, "expert"),
           "attention_held_out": held_out(att_rows, "attention")}
    if util_rows:
        rep["util_table"] = [[b, u] for _, b, u in util_rows]
    if args.bench:
        from paper_2504_02263_b200.pipeline import StageTimes, closed_form_total
        line = json.loads([ln for ln in open(args.bench) if ln.strip().startswith("{")][-1])
        c = line["config"]
        st = line.get("stage_times", {})
        b_e = c["b_a"] * c["n_a"] * model.topk * e_l // model.experts
        t_a, t_e = PM.attention_time(c["b_a"], cm), PM.expert_time(b_e, cm)
        m, L = c["m"], c["L_sim"]
        if c["n_a"] == 1 and c["n_e"] == 1 and "co-located" in c["workload"]:
            pred = m * L * (t_a + t_e)
        else:
            t_c = st.get("T_c_ms", 0.0) / 1e3
            pred = closed_form_total(StageTimes(t_a, t_e, t_c), m, L)
        rep["eq5_check"] = {"T_a_fit_ms": t_a * 1e3, "T_e_fit_ms": t_e * 1e3,
                            "predicted_ms": pred * 1e3, "measured_ms": line["ms_per_step"],
                            "measured_over_predicted": line["ms_per_step"] / (pred * 1e3)}
    print(json.dumps(rep), flush=True)


if __name__ == "__main__":
    main()
