"""Ping-pong timing model (SPEC.md:237-288 examples and invariants)."""

import random

import pytest

from paper_2504_02263_b200.pipeline import (StageTimes, closed_form_iter_bounds, closed_form_total,
                                            min_microbatches, simulate)


def test_min_microbatches_examples():
    assert min_microbatches(0.4, 1.0) == 3   # PAPER §4.1 "at least 3"
    assert min_microbatches(0.6, 1.0) == 4   # "at least 4"
    assert min_microbatches(0.0, 1.0) == 2
    assert min_microbatches(0.5, 1.0) == 3
    with pytest.raises(ValueError, match="not hideable"):
        min_microbatches(1.0, 1.0)


def test_eq5_example():
    t = StageTimes(1.0, 1.0, 0.0)
    assert closed_form_total(t, 3, 2) == 7
    assert closed_form_total(StageTimes(1, 2, 0.5), 1, 1) == 4


def test_simulator_matches_eq5_randomized():
    rng = random.Random(0)
    for _ in range(1000):
        ta, te = rng.uniform(0.1, 2), rng.uniform(0.1, 2)
        tf = max(ta, te)
        tc = rng.uniform(0, 0.95) * tf
        m = min_microbatches(tc, tf) + rng.randint(0, 2)
        L = rng.randint(1, 6)
        t = StageTimes(ta, te, tc)
        rep = simulate(t, m, L)
        ref = closed_form_total(t, m, L)
        if ta == te:  # Eq. 5 holds exactly for balanced stages
            assert abs(rep.total_latency - ref) <= 1e-9 * ref
        assert rep.total_latency <= ref * (1 + 1e-9)


def test_balanced_simulation_exact_and_bounds():
    rng = random.Random(1)
    for _ in range(300):
        tf = rng.uniform(0.1, 2)
        tc = rng.uniform(0, 0.95) * tf
        m = min_microbatches(tc, tf)
        L = rng.randint(1, 6)
        t = StageTimes(tf, tf, tc)
        rep = simulate(t, m, L)
        assert abs(rep.total_latency - closed_form_total(t, m, L)) <= 1e-9 * rep.total_latency
        lo, hi = closed_form_iter_bounds(t, m, L)
        assert lo - 1e-9 <= rep.iter_latency_per_microbatch <= hi + 1e-9


def test_timeline_structure():
    rep = simulate(StageTimes(1.0, 0.8, 0.3), 3, 4)
    for res in ("attention", "expert"):
        ev = sorted((r[4], r[5]) for r in rep.timeline if r[0] == res)
        assert all(a[1] <= b[0] + 1e-12 for a, b in zip(ev, ev[1:])), "resource overlap"
    phases = {(r[1], r[2], r[3]): (r[4], r[5]) for r in rep.timeline}
    for j in range(3):
        for l in range(4):
            a, d, f, c = (phases[(j, l, p)] for p in ("attn", "disp", "ffn", "comb"))
            assert a[1] <= d[0] + 1e-12 and d[1] <= f[0] + 1e-12 and f[1] <= c[0] + 1e-12
            if l:
                assert phases[(j, l - 1, "comb")][1] <= a[0] + 1e-12


def test_m1_expert_idle():
    t = StageTimes(1.0, 1.0, 0.25)
    rep = simulate(t, 1, 64)
    expect = (t.T_a + 2 * t.T_c) / (t.T_a + t.T_e + 2 * t.T_c)
    assert abs(rep.expert_idle_fraction - expect) < 0.01
