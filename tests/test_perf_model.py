"""Cost models -- the examples and properties the SPEC lists."""

import math
import random

import pytest

from paper_2504_02263_b200 import perf_model as PM
from paper_2504_02263_b200.config import ConfigError


def test_gemm_flops_examples():
    assert PM.gemm_flops(1, 1, 1) == 2
    assert PM.gemm_flops(156, 6144, 16384) == 2 * 156 * 6144 * 16384
    with pytest.raises(ConfigError):
        PM.gemm_flops(0, 6144, 16384)
    with pytest.raises(ConfigError):
        PM.gemm_flops(1 << 40, 1 << 20, 1 << 20)


def test_min_compute_bound_batch_examples():
    assert PM.min_compute_bound_batch(312e12, 2e12) == 156
    assert PM.min_compute_bound_batch(5.0, 5.0) == 1
    assert PM.min_compute_bound_batch(148e12, 4096e9) == 37


def test_ffn_utilization():
    assert PM.ffn_utilization(156, 312e12, 2e12, moe=(2, 8)) == pytest.approx(0.25)
    assert PM.ffn_utilization(0, 312e12, 2e12) == 0
    assert PM.ffn_utilization(1000, 312e12, 2e12) == 1.0
    prev = 0
    for b in range(0, 2000, 37):
        u = PM.ffn_utilization(b, 312e12, 2e12, moe=(2, 8))
        assert prev <= u <= 1
        prev = u


def test_affine_times_are_affine():
    cm = PM.CostModel(k1=2e-6, k2=1e-4, k3=3e-7, k4=5e-5)
    for a, b in [(0, 0), (3, 5), (100, 1000)]:
        assert PM.attention_time(a + b, cm) + PM.attention_time(0, cm) == pytest.approx(
            PM.attention_time(a, cm) + PM.attention_time(b, cm), rel=1e-15)
        assert PM.expert_time(a + b, cm) + PM.expert_time(0, cm) == pytest.approx(
            PM.expert_time(a, cm) + PM.expert_time(b, cm), rel=1e-15)
    assert PM.attention_time(0, cm) == cm.k2 and PM.expert_time(0, cm) == cm.k4
    cms = PM.CostModel(k1=2e-6, k2=0, k3=1e-7, k4=0, alpha=1e-9, beta=5e-7)
    assert PM.attention_time(10, cms, s=730) == pytest.approx(10 * (730e-9 + 5e-7))
    with pytest.raises(ConfigError):
        PM.CostModel(k1=0, k2=0, k3=1, k4=0)


def test_comm_time_examples():
    cm = PM.CostModel(k1=1, k2=0, k3=1, k4=0, util_curve=PM.UtilCurve(table=((1, 1.0),)))
    # symmetric: b_a*h*K/tp_a == b_e*h/tp_e, W equal -> volume / W
    t = PM.comm_time(128, 256, 6144, 2, 1, 1, 100e9, 100e9, cm)
    assert t == pytest.approx(128 * 6144 * 2 * 2 / 100e9)
    # Mixtral micro-batch 128, tp_a=2 -> per-pair payload 196,608 B (PAPER §7.3)
    assert 128 * 2 // 8 * 6144 * 2 // 2 == 196608
    # monotone: non-increasing in W, non-decreasing in b
    cm2 = PM.CostModel(k1=1, k2=0, k3=1, k4=0)
    base = PM.comm_time(64, 64, 4096, 2, 1, 1, 50e9, 50e9, cm2)
    assert PM.comm_time(64, 64, 4096, 2, 1, 1, 100e9, 50e9, cm2) <= base
    assert PM.comm_time(128, 64, 4096, 2, 1, 1, 50e9, 50e9, cm2) >= base
    # W_a -> inf: expert side decides
    t_inf = PM.comm_time(64, 64, 4096, 2, 1, 1, 1e30, 50e9, cm2)
    ve = 64 * 4096 * 2
    assert t_inf == pytest.approx(ve / (50e9 * cm2.util_curve(ve)))


def test_util_curve():
    u = PM.UtilCurve()
    assert u(65536) == pytest.approx(0.5)
    t = PM.UtilCurve.from_points([(1 << 20, 0.8), (1 << 14, 0.1), (1 << 16, 0.3), (1 << 18, 0.25)])
    assert t(1 << 14) == 0.1 and t(1 << 30) == 0.8 and t(1) == 0.1
    xs = [1 << k for k in range(10, 24)]
    us = [t(x) for x in xs]
    assert all(b >= a for a, b in zip(us, us[1:]))
    with pytest.raises(ConfigError):
        PM.UtilCurve(table=((1, 0.5), (2, 0.4)))


def test_calibrate_examples():
    f = PM.calibrate([(1, 3.0 + 0.5), (2, 6.0 + 0.5)], "expert")
    assert f.slope == pytest.approx(3.0) and f.intercept == pytest.approx(0.5)
    with pytest.raises(ConfigError):
        PM.calibrate([(4, 1.0), (4, 2.0)], "expert")
    with pytest.raises(ConfigError):
        PM.calibrate([(4, 1.0)], "attention")
    # noiseless affine data: machine precision
    rng = random.Random(0)
    for _ in range(20):
        k, c = rng.uniform(1e-7, 1e-5), rng.uniform(0, 1e-3)
        pts = [(b, k * b + c) for b in rng.sample(range(1, 5000), 6)]
        f = PM.calibrate(pts, "attention")
        assert f.slope == pytest.approx(k, rel=1e-9) and f.intercept == pytest.approx(c, rel=1e-7, abs=1e-15)


def test_calibrate_synthetic_memory_bound():
    """Memory-bound attention (KV traffic dominates): slope = bytes/token / BW."""
    h, g, s, bw = 6144, 8, 730, 6546.6e9
    pts = PM.synthetic_points("attention", [64, 128, 256, 512], h, 16384, 1e30, bw, seq_len=s, gqa_group=g)
    f = PM.calibrate(pts, "attention")
    assert f.slope == pytest.approx(2 * s * h * 2 / g / bw, rel=1e-6)
    # held-out prediction within 5%
    pe = PM.synthetic_points("expert", [256, 512, 1024, 2048, 4096], h, 16384, 1404.8e12, bw, c0=2e-5)
    fe = PM.calibrate(pe[::2], "expert")
    for b, t in pe[1::2]:
        assert abs(fe(b) - t) / t < 0.05


def test_profile_csv_roundtrip(tmp_path):
    p = tmp_path / "prof.csv"
    PM.write_profile(str(p), [("expert", 256, 1e-4), ("expert", 512, 1.8e-4), ("attention", 64, 2e-5),
                              ("attention", 128, 3.5e-5)], [("nvlink-peer", 65536, 0.2), ("nvlink-peer", 1 << 20, 0.7)])
    batch, util = PM.read_profile(str(p))
    assert batch["expert"] == [(256, 1e-4), (512, 1.8e-4)]
    assert util["nvlink-peer"][1] == (1 << 20, 0.7)
    cm = PM.cost_model_from_profile(str(p))
    assert cm.k3 == pytest.approx(8e-5 / 256) and cm.util_curve(1 << 20) == 0.7
    assert math.isclose(PM.attention_time(64, cm), 2e-5, rel_tol=1e-12)



def test_calibrate_tool_helpers(tmp_path):
    """calibrate.py's CPU-side pieces: the M2N JSONL -> UtilCurve rows and the
    held-out check (the GPU timing parts run on a B200 only)."""
    import json
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import calibrate as C

    p = tmp_path / "m2n.jsonl"
    recs = [{"T": t, "pair_bytes_avg": t * 49152.0, "ingress_bytes_busiest": t * 49152,
             "dispatch_only_p50_us": 20.0 + t * 0.1} for t in (1, 4, 64, 1024)]
    p.write_text("noise line\n" + "\n".join(json.dumps(r) for r in recs) + "\n")
    rows = C.util_from_m2n(str(p))
    assert [r[1] for r in rows] == [49152, 196608, 3145728, 50331648]
    assert all(0 < r[2] <= 1 for r in rows) and rows[-1][2] > rows[0][2]
    pts = [("expert", b, 1e-4 + 3e-7 * b) for b in (256, 512, 768, 1024, 1536, 2048)]
    h = C.held_out(pts, "expert")
    assert h["max_rel_err"] < 1e-9 and h["fit_on"] == [256, 768, 1536]
