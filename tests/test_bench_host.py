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
