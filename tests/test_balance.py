"""Expert load balancing (SPEC.md:397-414 examples and properties) and the
replicated-slot layout the runtime executes."""

import itertools

import numpy as np
import pytest

from oracle import oracle as O
from paper_2504_02263_b200 import balance as B


def test_node_cost_examples():
    assert B.node_cost([[1.0]], [5.0], 1.0).tolist() == [5.0]
    np.testing.assert_allclose(B.node_cost([[2 / 3, 1 / 3], [0, 1]], [3.0, 1.0], 1.0), [2.0, 2.0])
    # cold floor
    np.testing.assert_allclose(B.node_cost([[1, 0], [0, 1], [1, 0]], [0.1, 0.2, 0.3], 1.0), [2.0, 1.0])


def test_integral_two_experts():
    x = B.balance_experts([3.0, 1.0], 2, k_cold=1.0, mode="integral")
    assert sorted(B.node_cost(x, [3.0, 1.0], 1.0).tolist()) == [1.0, 3.0]


def test_fractional_is_water_filling():
    rng = np.random.default_rng(0)
    for _ in range(50):
        a = rng.random(rng.integers(1, 12)) * 10
        n = int(rng.integers(1, 6))
        x = B.balance_experts(a, n, mode="fractional")
        np.testing.assert_allclose(x.sum(1), 1.0, rtol=1e-12)
        c = B.node_cost(x, a)
        assert abs(c.max() - a.sum() / n) <= 1e-9 * max(a.sum(), 1)


def test_integral_lpt_bound_vs_brute_force():
    rng = np.random.default_rng(1)
    for _ in range(60):
        M, N = int(rng.integers(1, 9)), int(rng.integers(1, 4))
        a = rng.random(M) * 10
        x = B.balance_experts(a, N, mode="integral")
        assert ((x > 0).sum(1) == 1).all()
        greedy = B.node_cost(x, a).max()
        best = min(max(sum(a[i] for i in range(M) if asg[i] == j) for j in range(N))
                   for asg in itertools.product(range(N), repeat=M))
        assert greedy <= 4 / 3 * best + 1e-9


def test_replicated_bounds_and_row_stochastic():
    """row-stochastic placements; greedy within the trivial
    bound max(max_i a_i, 2 * Sum/N); on skewed loads replication helps on average."""
    rng = np.random.default_rng(2)
    ratios = []
    for _ in range(200):
        a = rng.pareto(1.5, int(rng.integers(2, 17))) + 0.01
        n = int(rng.integers(2, 5))
        xi = B.balance_experts(a, n, mode="integral")
        xr = B.balance_experts(a, n, mode="replicated", max_replicas=2)
        np.testing.assert_allclose(xr.sum(1), 1.0)
        assert ((xr > 0).sum(1) <= 2).all()
        for x in (xi, xr):
            assert B.node_cost(x, a).max() <= max(a.max(), 2 * a.sum() / n) + 1e-9
        ratios.append(B.node_cost(xr, a).max() / B.node_cost(xi, a).max())
    assert np.mean(ratios) < 1.0


def test_slots_from_placement():
    loads = np.array([40.0, 5, 5, 5, 30, 5, 5, 5])
    sl = B.balanced_slots(loads, 2, max_replicas=2)
    assert sl.P == 2 * sl.P_l and sl.E == 8
    for e in range(8):
        c = sl.rep[e, 0]
        assert 1 <= c <= 2
        for r in range(c):
            assert sl.phys2log[sl.rep[e, 1 + r]] == e
    assert set(np.flatnonzero(sl.phys2log >= 0).tolist()) == {int(p) for e in range(8) for p in sl.rep[e, 1:1 + sl.rep[e, 0]]}
    # balancing lowers the expected max GPU load vs the contiguous default
    ident = B.identity_slots(8, 2)
    assert sl.expected_gpu_rows(loads).max() < ident.expected_gpu_rows(loads).max()


def test_physical_slot_rule_splits_evenly():
    rep = np.array([[2, 3, 7], [1, 1, 0], [1, 2, 0], [1, 0, 0]], np.int32)  # expert 0 on slots 3 and 7
    idx = np.zeros((101, 1), np.int32)
    for s in range(3):
        p = O.physical_slots(idx, rep, s)
        n3, n7 = (p == 3).sum(), (p == 7).sum()
        assert abs(n3 - n7) <= 1 and n3 + n7 == 101


def test_oracle_replicated_layer_equals_unreplicated():
    """Replicas run the same weights: outputs are identical to the plain layer."""
    wts = O.synth_weights(512, 256, 8, seed=0)
    xs = [O.synth_tokens(40, 512, seed=3), O.synth_tokens(23, 512, seed=4)]
    plain = O.moe_layer(xs, wts, 2, n_e=2)
    sl = B.balanced_slots(np.array([20.0, 1, 1, 1, 15, 1, 1, 1]), 2)
    rep = O.moe_layer(xs, wts, 2, n_e=2, rep=sl.rep, phys2log=sl.phys2log)
    for s in range(2):
        np.testing.assert_array_equal(rep.idx[s], plain.idx[s])
        np.testing.assert_array_equal(rep.out[s], plain.out[s])
        np.testing.assert_array_equal(sl.phys2log[rep.pidx[s]], plain.idx[s])
    assert rep.cnt.sum() == plain.cnt.sum()


def test_identity_slots_match_default_layout():
    sl = B.identity_slots(8, 2)
    assert sl.P_l == 4 and sl.logical_of_local(1) == [4, 5, 6, 7]
    with pytest.raises(ValueError):
        B.identity_slots(8, 3)


def test_spread_slots_balances_non_dividing_counts():
    """8 experts on 3, 5 or 6 expert GPUs: every GPU carries E / n_e experts'
    rows under the (t + s) mod nrep replica rule; 8 on 4 is the identity."""
    from paper_2504_02263_b200.balance import identity_slots, spread_slots
    for n_e, P_l in ((3, 4), (5, 4), (6, 3), (7, 2)):
        sl = spread_slots(8, n_e)
        assert sl.P_l == P_l and sl.P == n_e * P_l
        rows = sl.expected_gpu_rows(np.ones(8))
        np.testing.assert_allclose(rows, 8 / n_e)
        assert set(sl.phys2log[sl.phys2log >= 0]) == set(range(8))
        # the replica rule spreads a replicated expert's tokens evenly
        for e in range(8):
            c = int(sl.rep[e, 0])
            t = np.arange(600)
            for s in range(3):
                got = np.bincount((t + s) % c, minlength=c)
                assert got.max() - got.min() <= 1
    ident = spread_slots(8, 4)
    assert ident.P == identity_slots(8, 4).P and (ident.phys2log == np.arange(8)).all()


# ---------------- attention batch composition ----------------
def _cm(alpha=2e-9, beta=1e-7, k2=3e-5):
    from paper_2504_02263_b200.perf_model import CostModel
    return CostModel(k1=alpha * 730 + beta, k2=k2, k3=1e-6, k4=1e-4, alpha=alpha, beta=beta)


def test_compose_identical_requests_equal_nodes():
    cm = _cm()
    for n_a, per in ((4, 3), (3, 5), (2, 64)):
        reqs = [(i, 730) for i in range(n_a * per)]
        plan = B.compose_attention_batches(reqs, n_a, cm)
        assert [len(a) for a in plan.assignment] == [per] * n_a
        assert max(plan.predicted) - min(plan.predicted) <= 1e-12 * max(plan.predicted)


def test_compose_giant_request_isolated():
    cm = _cm()
    reqs = [(0, 10), (1, 12), (2, 100000), (3, 9), (4, 11), (5, 10), (6, 8)]
    plan = B.compose_attention_batches(reqs, 3, cm)
    giant = [a for a in plan.assignment if 2 in a]
    assert giant == [[2]]


def test_compose_assigns_every_request_once_and_is_deterministic():
    cm = _cm()
    rng = np.random.default_rng(1)
    reqs = [(int(i), int(s)) for i, s in zip(rng.permutation(200), rng.integers(1, 1460, 200))]
    p1 = B.compose_attention_batches(reqs, 6, cm)
    p2 = B.compose_attention_batches(reqs, 6, cm)
    assert p1.assignment == p2.assignment
    ids = sorted(r for a in p1.assignment for r in a)
    assert ids == sorted(r for r, _ in reqs)
    # predicted = k2 + sum of costs, per node
    length = dict(reqs)
    for ids_j, t in zip(p1.assignment, p1.predicted):
        assert t == pytest.approx(cm.k2 + sum(B.request_cost(length[r], cm) for r in ids_j), rel=1e-12)
    # seq_lens view for the attention stage
    lens = p1.seq_lens(reqs)
    assert [len(v) for v in lens] == [len(a) for a in p1.assignment]


def test_compose_max_batch_caps_bins():
    cm = _cm()
    reqs = [(i, 100 + i) for i in range(12)]
    plan = B.compose_attention_batches(reqs, 3, cm, target_time=1.0, max_batch=4)  # huge target: first-fit
    assert [len(a) for a in plan.assignment] == [4, 4, 4]
    with pytest.raises(ValueError):
        B.compose_attention_batches(reqs, 2, cm, max_batch=5)


def test_compose_near_brute_force_optimum():
    """random seq lens, n_a = 4, <= 8 requests: max/min predicted node time
    within the brute-force optimal ratio + 15 %."""
    cm = _cm(k2=0.0)
    rng = np.random.default_rng(7)
    for trial in range(40):
        n = int(rng.integers(4, 9))
        lens = rng.integers(1, 1460, n)
        reqs = list(enumerate(lens.tolist()))
        plan = B.compose_attention_batches(reqs, 4, cm)
        got = max(plan.predicted) / min(plan.predicted)
        cost = [B.request_cost(s, cm) for s in lens]
        best = np.inf
        for assign in itertools.product(range(4), repeat=n):
            if len(set(assign)) < 4:
                continue
            t = np.zeros(4)
            for i, j in enumerate(assign):
                t[j] += cost[i]
            best = min(best, t.max() / t.min())
        assert got <= best * 1.15 + 1e-12, (trial, got, best)


def test_compose_lpt_with_equal_batches():
    """mode='lpt' + max_batch: equal request counts per node and balanced
    predicted times (the bench's per-GPU micro-batches)."""
    cm = _cm()
    rng = np.random.default_rng(3)
    reqs = list(enumerate(rng.integers(1, 1460, 3 * 512).tolist()))
    plan = B.compose_attention_batches(reqs, 3, cm, max_batch=512, mode="lpt")
    assert [len(a) for a in plan.assignment] == [512] * 3
    assert max(plan.predicted) / min(plan.predicted) < 1.001
    with pytest.raises(ValueError):
        B.compose_attention_batches(reqs, 3, cm, mode="best")
