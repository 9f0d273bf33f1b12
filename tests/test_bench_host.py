"""Host-side logic of bench.py (no GPU): the layout choice at each GPU count
and the M2N link-byte accounting behind `m2n.roofline`."""

import bench


def test_choose_split_planner_picks_colocation_for_8x22b():
    assert bench.choose_split(1, "mixtral-8x22b", "planner")[:3] == (1, 1, True)
    for n in (2, 4, 8):
        n_a, n_e, colo, src, tp = bench.choose_split(n, "mixtral-8x22b", "planner")
        assert tp == 1
        assert (n_a, n_e, colo) == (n, n, True)
        assert src.startswith("planner.search_box")


def test_choose_split_config_and_overrides():
    assert bench.choose_split(8, "mixtral-8x22b", "config")[:3] == (6, 2, False)
    assert bench.choose_split(4, "mixtral-8x22b", "config")[:3] == (3, 1, False)
    assert bench.choose_split(4, "mixtral-8x22b", "planner", split="2+2")[:3] == (2, 2, False)
    assert bench.choose_split(4, "mixtral-8x22b", "planner", split="2+2", tp_e=2)[4] == 2
    assert bench.choose_split(4, "dbrx", "planner", colocated=True)[:3] == (4, 4, True)
    # no calibration for this shape: the BASELINE config split
    assert bench.choose_split(4, "dbrx", "planner")[3] == "BASELINE.json config split"


def test_m2n_leg_bytes():
    H = 6144
    # co-located 2 GPUs: diagonal rows stay local
    leg1, leg2, off = bench.m2n_leg_bytes([[3000, 3004], [3029, 3100]], H)
    assert off == [[0, 3004], [3029, 0]]
    assert leg1 == 3029 * (2 * H + 8) and leg2 == 3029 * 2 * H
    # disaggregated 3+1: the expert GPU (rank 3) receives every row
    mat = [[0, 0, 0, 2048], [0, 0, 0, 2048], [0, 0, 0, 2048], [0, 0, 0, 0]]
    leg1, leg2, _ = bench.m2n_leg_bytes(mat, H)
    assert leg1 == 6144 * (2 * H + 8) and leg2 == 6144 * 2 * H


def test_reference_arm_runs_whole_layer_and_reports_bench_config():
    """--impl reference times the oracle's whole layer per step (no
    projection): ms_per_step x steps fits the wall time, and its config is
    bench_config() -- the dict the GPU arm prints."""
    import json
    import os
    import subprocess
    import sys
    import types

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--shape", "tiny",
                          "--b-a", "32", "--steps", "2", "--warmup", "1"], capture_output=True, text=True,
                         timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["steps"] == 2
    assert line["ms_per_step"] * line["steps"] / 1e3 <= line["wall_s"]
    assert "no sampling" in line["cpu_baseline"]["sample"]
    from paper_2504_02263_b200.config import as_model_spec
    args = types.SimpleNamespace(layers=4, merge=True, attn="real", graph=True)
    want = bench.bench_config(args, as_model_spec("tiny"), 1, 1, True, "1 GPU: co-located", 1, 1, 96, 1)
    assert line["config"] == want


def test_disaggregated_layout_for_the_pingpong_line():
    import argparse

    args = argparse.Namespace(shape="mixtral-8x22b", m=3, b_a=1024)
    # expert share of the per-token GPU time ~0.65 (T_e 3.3 ms vs T_a 1.8 ms per merged micro-batch)
    (n_a, n_e, colo, src, tp, model, m, b_a), slots = bench.disaggregated_layout(args, 8, 0.65)
    assert (n_a, n_e, colo, tp, m, b_a) == (3, 5, False, 1, 3, 1024)
    assert slots is not None and slots.n_e == 5 and slots.P % 5 == 0  # 8 experts over 5 GPUs
    assert "3+5" in src
    (n_a, n_e, *_), slots = bench.disaggregated_layout(args, 4, 0.65)
    assert (n_a, n_e) == (2, 2) and slots is None  # min(2/0.35, 2/0.65) > min(1/0.35, 3/0.65)
    (n_a, n_e, *_), slots = bench.disaggregated_layout(args, 4, 0.70)
    assert (n_a, n_e) == (1, 3) and slots.P == 12  # 1+3 wins from s = 2/3
    (n_a, n_e, *_), slots = bench.disaggregated_layout(args, 2, 0.65)
    assert (n_a, n_e) == (1, 1) and slots is None
    (n_a, n_e, *_), slots = bench.disaggregated_layout(args, 8, 0.99)  # at least one attention GPU
    assert (n_a, n_e) == (1, 7)


def test_pingpong_summary_keeps_the_comparable_fields():
    sub = {"value": 1.0, "value_per_gpu": 0.5, "ms_per_step": 3.0, "stage_times": {"T_a_ms": 1}, "clocks": {},
           "gpu_launches": 7, "attention": None, "config": {"n_a": 1}, "roofline": {"achieved": 900.0, "frac": 0.6},
           "parity": {"routing_bit_exact": True, "combine_bit_exact": True}, "e2e": None}
    out = bench.pingpong_summary(sub, 0.6)
    assert out["value"] == 1.0 and out["expert_ffn"]["achieved"] == 900.0 and out["parity"]["routing_bit_exact"]
    assert "e2e" not in out and bench.pingpong_summary(None, 0.5) is None


def test_plan_json_with_attention_tp_reaches_the_bench(tmp_path):
    """A plan file whose DeploymentPlan has tp_a = 2 round-trips through
    save_plan / load_plan, and bench.py --plan-json takes tp_a from it."""
    import argparse

    from paper_2504_02263_b200.config import (Catalog, ConfigBundle, DeploymentPlan, SearchLimits, WorkloadSpec,
                                               as_model_spec, b200_gpu, load_plan, save_plan)

    bundle = ConfigBundle(Catalog([b200_gpu()]), as_model_spec("mixtral-8x22b"), WorkloadSpec(), SearchLimits())
    dp = DeploymentPlan(n_a=2, n_e=2, m=2, b_a=512, tp_a=2)
    out = tmp_path / "plan.json"
    save_plan(bundle, dp, out)
    assert load_plan(out)[1] == dp
    args = argparse.Namespace(plan_json=str(out), shape="dbrx", m=3, b_a=1024, tp_a=1)
    n_a, n_e, colo, src, tp_e = bench.apply_plan_json(args)
    assert (n_a, n_e, colo, tp_e, args.tp_a, args.m, args.b_a) == (2, 2, False, 1, 2, 2, 512)


def test_reference_arm_under_torchrun_uses_the_host_threads():
    """torchrun sets OMP_NUM_THREADS=1 in every rank; the reference arm's
    rank 0 must still run the CPU oracle on all host threads (else the N > 1
    reference runs are ~30x slower than the N = 1 one), and the other ranks
    exit 0 without work."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    probe = ("import os, sys; sys.argv = ['bench.py'] + sys.argv[1:]; "
             "exec(open('bench.py').read().split('import numpy as np')[0]); print(os.environ['OMP_NUM_THREADS'])")
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", OMP_NUM_THREADS="1")
    out = subprocess.run([sys.executable, "-c", probe, "--impl", "reference", "--gpus", "2"], env=env, cwd=root,
                         capture_output=True, text=True, check=True).stdout.strip()
    assert out == str(len(os.sched_getaffinity(0)))
    out = subprocess.run([sys.executable, "-c", probe, "--gpus", "2"], env=env, cwd=root,
                         capture_output=True, text=True, check=True).stdout.strip()
    assert out == "1"  # the GPU arm is left alone
    env["RANK"] = "1"
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2"], env=env, cwd=root,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and not r.stdout.strip()
