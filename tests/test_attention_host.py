"""Host-side logic of the attention stage (paper_2504_02263_b200/attention.py):
head layout, batch composition, paged-KV block tables (CPU tensors; the
kernels themselves are covered by tests/test_gpu_attention.py)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2504_02263_b200 import attention as A  # noqa: E402
from paper_2504_02263_b200.config import BENCH_SHAPES, MoeModelSpec  # noqa: E402


def test_head_layout_matches_spec_kv_width():
    """n_kv * 128 = h / g: the KV bytes per token the SPEC's 2 b s h / g counts."""
    for name in ("mixtral-8x22b", "mixtral-8x7b", "dbrx", "deepseek-v3"):
        m = BENCH_SHAPES[name]
        nh, nkv = A.head_layout(m)
        assert nh == m.hidden // 128 and nh % nkv == 0
        assert nkv * 128 == m.hidden // m.gqa_group
    assert A.head_layout(BENCH_SHAPES["tiny"]) == (4, 1)  # g clamped to the head count
    with pytest.raises(ValueError):
        A.head_layout(MoeModelSpec("odd", layers=1, hidden=200, intermediate=256, experts=2, topk=1))


def test_batch_composition():
    c = A.batch_composition(20000, 730, seed=1)
    assert c.min() >= 1 and c.max() <= 2 * 730 - 1
    assert abs(c.mean() - 730) < 10
    assert (A.batch_composition(7, 730, mode="fixed") == 730).all()
    np.testing.assert_array_equal(A.batch_composition(50, 730, seed=3), A.batch_composition(50, 730, seed=3))


def test_paged_cache_block_table_is_a_permutation():
    ctx = np.array([0, 1, 63, 64, 65, 700, 1459], np.int32)
    c = A.PagedKVCache(len(ctx), 2, ctx, layers=2, device="cpu", seed=4, headroom=64, fill=False)
    need = (ctx + 1 + 64 + 63) // 64
    assert c.max_pages == need.max() and c.num_pages == need.sum()
    used = np.concatenate([c.block_table_host[t, : need[t]] for t in range(len(ctx))])
    assert sorted(used.tolist()) == list(range(c.num_pages))  # every page owned exactly once
    assert c.k[0].shape == (c.num_pages, 2, 64, 128) and len(c.v) == 2
    assert c.kv_bytes_read() == int((ctx + 1).sum()) * 2 * 128 * 2 * 2
    np.testing.assert_array_equal(c.lens.numpy(), ctx + 1)
    c.advance()
    np.testing.assert_array_equal(c.pos.numpy(), ctx + 1)
    tight = A.PagedKVCache(1, 1, np.array([63], np.int32), layers=1, device="cpu", fill=False)
    with pytest.raises(RuntimeError):
        tight.advance()  # 64 tokens fill the only page; a 65th would need another


def test_request_cost_model_and_composed_batches():
    """Per-request attention cost alpha * seq_len + beta from the KV bytes at the
    HBM rate and the projection FLOPs at the tensor rate; composed batches
    over the DP attention GPUs have b_a requests each and near-equal predicted
    times, identical on every rank for a seed."""
    m = BENCH_SHAPES["mixtral-8x22b"]
    cm = A.request_cost_model(m, hbm_gbs=6500.0, tflops=1400.0)
    nh, nkv = A.head_layout(m)
    assert cm.alpha == pytest.approx(2 * nkv * 128 * 2 / 6.5e12)
    assert cm.beta == pytest.approx(2.0 * m.hidden * (nh + 2 * nkv + nh) * 128 / 1.4e15)
    lens, plan = A.composed_ctx_lens(m, 3, 512, 730, seed=4)
    assert [len(v) for v in lens] == [512] * 3
    assert max(plan.predicted) / min(plan.predicted) < 1.001
    lens2, _ = A.composed_ctx_lens(m, 3, 512, 730, seed=4)
    assert all((a == b).all() for a, b in zip(lens, lens2))
    pool = np.sort(A.batch_composition(3 * 512, 730, 4))
    assert (np.sort(np.concatenate(lens)) == pool).all()  # every request exactly once
