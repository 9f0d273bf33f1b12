"""Deployment-plan search (Algorithm 1; SPEC.md:305-344 examples and properties)."""

import dataclasses
import random

import pytest

from paper_2504_02263_b200 import perf_model as PM
from paper_2504_02263_b200 import planner as PL
from paper_2504_02263_b200.config import GpuSpec, MoeModelSpec, SearchLimits, WorkloadSpec, b200_gpu

GB = 1e9


def _cm(k1=2e-6, k2=1e-4, k3=4e-7, k4=3e-4):
    return PM.CostModel(k1=k1, k2=k2, k3=k3, k4=k4)


MIXTRAL = MoeModelSpec("Mixtral-8x22B", layers=56, hidden=6144, intermediate=16384, experts=8, topk=2)


def test_balance_attention_nodes_examples():
    assert PL.balance_attention_nodes(PM.CostModel(k1=2, k2=0, k3=1, k4=0), 8, 2) == 8
    assert PL.balance_attention_nodes(PM.CostModel(k1=1, k2=0, k3=1, k4=0), 4, 4) == 1
    assert PL.balance_attention_nodes(PM.CostModel(k1=1.5, k2=0, k3=1, k4=0), 16, 4) == 6


def test_param_sizes_pin():
    # Mixtral-8x22B P_e = 22,548,578,304 bytes
    assert PL.param_sizes(MIXTRAL)[1] == 22_548_578_304
    assert PL.param_sizes(MIXTRAL, swiglu=True)[1] == 22_548_578_304 * 3 // 2


def test_max_batch_is_maximal():
    """Returned B is feasible and B + m n_a is not (linear-scan oracle)."""
    rng = random.Random(0)
    gpu = b200_gpu()
    found = 0
    for _ in range(25):
        cm = _cm(k1=rng.uniform(1e-7, 5e-6), k2=rng.uniform(0, 3e-4), k3=rng.uniform(1e-8, 1e-6),
                 k4=rng.uniform(0, 5e-4))
        wl = WorkloadSpec(slo_tbt=rng.uniform(0.02, 0.3))
        n_a, m = rng.randint(1, 4), rng.randint(2, 4)
        p, _ = PL.max_batch_under_slo(MIXTRAL, gpu, gpu, cm, wl, 1, 1, n_a, 2, m, b_max=1 << 16,
                                      balance_slack=float("inf"), colocated=False, swiglu=True,
                                      expert_nodes_hold=4)
        step = m * n_a
        feas = [k * step for k in range(1, (1 << 16) // step + 1)
                if PL.evaluate(MIXTRAL, gpu, gpu, cm, wl, 1, 1, n_a, 2, m, k * step, balance_slack=float("inf"),
                               swiglu=True, expert_nodes_hold=4)[0] is not None]
        if p is None:  # SLO / memory bind at every B, or a lower constraint binds at the largest B
            continue
        found += 1
        assert p.B % step == 0
        assert PL.evaluate(MIXTRAL, gpu, gpu, cm, wl, 1, 1, n_a, 2, m, p.B, balance_slack=float("inf"),
                           swiglu=True, expert_nodes_hold=4)[0] is not None
        assert PL.evaluate(MIXTRAL, gpu, gpu, cm, wl, 1, 1, n_a, 2, m, p.B + step, balance_slack=float("inf"),
                           swiglu=True, expert_nodes_hold=4)[0] is None
        assert p.B == max(feas)
    assert found >= 10


def _brute(model, gpu_a, gpu_e, cm, wl, limits, slack):
    best = None
    p_a, p_e = PL.param_sizes(model)
    for tp_e in [t for t in PL.TP_CHOICES if t <= gpu_e.max_gpus_per_node]:
        for tp_a in [t for t in PL.TP_CHOICES if t <= gpu_a.max_gpus_per_node]:
            if not (tp_a * gpu_a.mem_capacity > p_a and tp_e * gpu_e.mem_capacity > p_e):
                continue
            cmt = PL._tp_scaled(cm, tp_a, tp_e)
            n_a = PL.balance_attention_nodes(cmt, model.experts, model.topk)
            for m in range(3, limits.max_microbatches + 1):
                p, _ = PL.max_batch_under_slo(model, gpu_a, gpu_e, cmt, wl, tp_a, tp_e, n_a, model.experts, m,
                                              balance_slack=slack)
                if p is not None and (best is None or p.tpuc > best.tpuc or
                                      (p.tpuc == best.tpuc and (p.gpus, p.m, p.tp_a) < (best.gpus, best.m, best.tp_a))):
                    best = p
    return best


def test_search_equals_brute_force_and_invariants():
    gpu = GpuSpec("G", price=2.0, mem_capacity=80 * GB, mem_bandwidth=2e12, compute=312e12,
                  net_bandwidth_per_gpu=25e9, max_power=400.0, max_gpus_per_node=8)
    cm = _cm(k1=1e-6, k2=5e-5, k3=2.5e-7, k4=1e-4)
    wl = WorkloadSpec(slo_tbt=0.15)
    lim = SearchLimits(max_microbatches=4)
    p = PL.search(MIXTRAL, gpu, gpu, cm, wl, lim, balance_slack=0.5)
    b = _brute(MIXTRAL, gpu, gpu, cm, wl, lim, 0.5)
    assert p and b and p.tpuc == b.tpuc and (p.tp_a, p.tp_e, p.m, p.B) == (b.tp_a, b.tp_e, b.m, b.B)
    # scale invariance of prices
    gpu2 = dataclasses.replace(gpu, price=7.0)
    p2 = PL.search(MIXTRAL, gpu2, gpu2, cm, wl, lim, balance_slack=0.5)
    assert (p2.tp_a, p2.tp_e, p2.m, p2.B) == (p.tp_a, p.tp_e, p.m, p.B)
    # relaxing the SLO never lowers the best tpuc
    p3 = PL.search(MIXTRAL, gpu, gpu, cm, WorkloadSpec(slo_tbt=0.3), lim, balance_slack=0.5)
    assert p3.tpuc >= p.tpuc
    # every returned plan re-checks feasible
    assert p.T_iter_upper <= wl.slo_tbt and p.T_c < p.T_f


def test_search_infeasible_memory():
    tiny_gpu = GpuSpec("small", price=1.0, mem_capacity=1 * GB, mem_bandwidth=1e12, compute=1e14,
                       max_gpus_per_node=8)
    r = PL.search(MIXTRAL, tiny_gpu, tiny_gpu, _cm(), WorkloadSpec())
    assert not r and all("memory" in why for _, why in r.reasons)


def test_search_box_b200():
    """The 8-GPU box search returns a feasible split with the calibrated
    Mixtral-8x22B coefficients (profiles/r01_calibration_8x22b.json values)."""
    cm = PM.CostModel(k1=3.0956e-07, k2=1.0e-05, k3=4.4384e-07, k4=3.2245e-04,
                      util_curve=PM.UtilCurve.from_points([(196608, 0.0084), (3145728, 0.12), (50331648, 0.58)]))
    table = []
    p = PL.search_box(MIXTRAL, b200_gpu(), PL.cm_scaled_for_experts(cm, 8), WorkloadSpec(), 8, explain=table)
    assert p and p.gpus == 8 and p.T_iter_upper <= 0.150
    assert len(table) >= 4
    assert any(r["colocated"] for r in table)
    assert any(r["tp_e"] == 2 and not r["colocated"] for r in table)  # expert-TP layouts are candidates


def test_plan_json_round_trip(tmp_path):
    """Plan JSON output: the planner CLI writes the
    config + plan section, load_plan reads back the same DeploymentPlan, and
    bench.py's --plan-json takes its layout from it."""
    import argparse
    import json
    import os

    import bench
    from paper_2504_02263_b200.config import load_plan

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "plan.json"
    rc = PL.main(["--calibration", os.path.join(root, "profiles", "r01_calibration_8x22b.json"),
                  "--gpus", "4", "--b-a", "1024", "--out", str(out)])
    assert rc == 0
    bundle, plan = load_plan(out)
    assert (plan.n_a, plan.n_e, plan.colocated, plan.b_a) == (4, 4, True, 1024)
    assert bundle.model.name == MIXTRAL.name
    assert "tpuc" in json.loads(out.read_text())["plan_info"]
    args = argparse.Namespace(plan_json=str(out), shape="tiny", m=3, b_a=64)
    n_a, n_e, colo, src, tp = bench.apply_plan_json(args)
    assert (n_a, n_e, colo, tp, args.m, args.b_a) == (4, 4, True, 1, 1, 1024)
    assert args.shape.name == MIXTRAL.name and src.startswith("--plan-json")


def test_search_box_attention_tp_candidates_and_deployment():
    """Attention TP: the box search evaluates attention nodes of
    tp_a GPUs (tp_a must divide the KV heads), and to_deployment maps a node's
    batch onto its GPUs' shards (b_a per GPU = node batch / tp_a)."""
    from paper_2504_02263_b200.config import DeploymentPlan

    cm = PM.CostModel(k1=3.0956e-07, k2=1.0e-05, k3=4.4384e-07, k4=3.2245e-04,
                      util_curve=PM.UtilCurve.from_points([(196608, 0.0084), (3145728, 0.12), (50331648, 0.58)]))
    table = []
    PL.search_box(MIXTRAL, b200_gpu(), PL.cm_scaled_for_experts(cm, 8), WorkloadSpec(), 8, explain=table)
    tpa = {r["tp_a"] for r in table if not r["colocated"]}
    assert {1, 2} <= tpa and 4 not in tpa  # Mixtral-8x22B has 6 KV heads: tp_a in {1, 2} of (1, 2, 4)
    p = PL.Plan(tp_a=2, tp_e=1, n_a=1, n_e=2, m=2, B=4096, b_a=2048.0, b_e=2048.0, T_a=1e-3, T_e=1e-3, T_c=1e-4,
                T_f=1e-3, T_iter_upper=0.1, T_total=0.1, tpuc=1.0, gpus=4)
    d = PL.to_deployment(p)
    assert d == DeploymentPlan(n_a=2, n_e=2, m=2, b_a=1024, tp_a=2)
