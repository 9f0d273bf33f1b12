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
