"""The CPU oracle, pinned before it is trusted.

The reference has no tests or golden vectors for this path, so
the oracle is pinned by (1) the sizing numbers the reference does state,
(2) known-answer constructions whose result is exact by hand, (3) an
independent float64 evaluation, and (4) the committed regression fixtures in
tests/golden/ (make_golden.py).
"""

import hashlib
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------ reference pins ----
def test_pair_payload_bytes_paper_example():
    # PAPER.md:632 / SPEC.md:172: Mixtral, micro-batch 128, tp_a = 2 -> 196,608 B
    assert O.pair_payload_bytes(128, 2, 8, 6144, tp_a=2) == 196608


def test_gemm_flops_spec_example():
    # SPEC.md:120-128 defines gemm_flops = 2*b*h_in*h_out and quotes the example
    # (156, 6144, 16384) as 31,407,899,148,288 (~3.14e13).  That number does not
    # follow from its own formula (2*156*6144*16384 = 31,406,948,352 ~ 3.14e10);
    # the formula is the contract, the quoted digits are a SPEC typo.
    assert O.gemm_flops(156, 6144, 16384) == 2 * 156 * 6144 * 16384 == 31_406_948_352
    assert O.gemm_flops(156, 6144, 16384) != 31_407_899_148_288
    assert O.gemm_flops(1, 1, 1) == 2
    with pytest.raises(ValueError):
        O.gemm_flops(0, 1, 1)


def test_expert_param_bytes_spec_example():
    assert O.expert_param_bytes(56, 6144, 16384) == 22_548_578_304  # SPEC.md:153 (2 GEMMs)
    assert O.expert_param_bytes(56, 6144, 16384, swiglu=True) == 22_548_578_304 * 3 // 2


# ------------------------------------------------------- known answers ----
def test_det_expf_accuracy():
    for d in np.concatenate([np.linspace(-87, 0, 2001), [-1e-8, -0.5, -0.6931472, -20.0]]):
        got = O.det_expf(float(np.float32(d)))
        ref = math.exp(float(np.float32(d)))
        assert abs(got - ref) <= 2.5e-7 * ref + 1e-44
    assert O.det_expf(0.0) == 1.0
    assert O.det_expf(-100.0) == 0.0
    assert O.det_expf(float("nan")) == 0.0


def test_router_one_hot_tokens_exact():
    """x = one-hot rows: logit[t, e] == wg[e, i_t] exactly; top-K by hand."""
    H, E, K = 512, 8, 3
    wg = O.synth_weights(H, 128, E, seed=3, experts=[]).wg
    pos = np.arange(0, H, 37)[:13]
    x = np.zeros((len(pos), H), np.uint16)
    x[np.arange(len(pos)), pos] = 0x3F80  # bf16 1.0
    idx, w, lg = O.router(x, wg, K, want_logits=True)
    col = O.bf16_to_f32(wg)[:, pos].T
    np.testing.assert_array_equal(lg, col)
    for t in range(len(pos)):
        order = sorted(range(E), key=lambda e: (-col[t, e], e))[:K]
        assert list(idx[t]) == order
        ex = np.exp(col[t, order].astype(np.float64) - col[t, order[0]])
        np.testing.assert_allclose(w[t], ex / ex.sum(), rtol=1e-6)


def test_router_ties_lower_index():
    x = O.synth_tokens(5, 256, seed=1)
    wg = np.zeros((6, 256), np.uint16)
    idx, w = O.router(x, wg, 4)
    assert (idx == np.arange(4)).all() and (w == np.float32(0.25)).all()


def test_router_against_float64():
    """Independent evaluation: top-K equals float64 argsort wherever the K-th /
    (K+1)-th gap exceeds fp32 reduction noise; weights within 1e-6."""
    T, H, E, K = 256, 4096, 16, 4
    x = O.synth_tokens(T, H, seed=2)
    wg = O.synth_weights(H, 128, E, seed=4, experts=[]).wg
    idx, w, lg = O.router(x, wg, K, want_logits=True)
    ref = O.bf16_to_f32(x).astype(np.float64) @ O.bf16_to_f32(wg).astype(np.float64).T
    assert np.abs(lg - ref).max() < 1e-5
    srt = np.sort(ref, axis=1)[:, ::-1]
    clear = (srt[:, K - 1] - srt[:, K]) > 1e-4
    ref_idx = np.argsort(-ref, axis=1, kind="stable")[:, :K]
    assert clear.mean() > 0.9
    np.testing.assert_array_equal(idx[clear], ref_idx[clear])
    sel = np.take_along_axis(ref, idx.astype(np.int64), 1)
    ex = np.exp(sel - sel[:, :1])
    np.testing.assert_allclose(w, ex / ex.sum(1, keepdims=True), rtol=2e-6, atol=1e-7)


def test_place_invariants():
    rng = np.random.default_rng(0)
    T, K, E = 300, 4, 16
    idx = np.stack([rng.choice(E, K, replace=False) for _ in range(T)]).astype(np.int32)
    cnt, slot = O.place(idx, E)
    assert cnt.sum() == T * K
    for e in range(E):
        t, k = np.nonzero(idx == e)
        assert sorted(slot[t, k]) == list(range(cnt[e]))
        assert (np.diff(slot[t, k][np.argsort(t)]) == 1).all()  # ascending token order


def test_dispatch_layout_invariants():
    """Receive rows: distinct per expert GPU, inside region (e_l, s) of cap_s
    rows, and dense from the region start (slots 0..cnt-1); the virtual
    order of the expert GEMM is 128-row aligned per expert."""
    rng = np.random.default_rng(1)
    n_a, T, K, E, n_e = 3, 100, 2, 8, 2
    E_l = E // n_e
    idxs = [np.stack([rng.choice(E, K, replace=False) for _ in range(T)]).astype(np.int32) for _ in range(n_a)]
    pl = [O.place(i, E) for i in idxs]
    cnt = np.stack([c for c, _ in pl])
    layout = O.dispatch_layout(cnt, E_l)
    seen = {q: set() for q in range(n_e)}
    for s in range(n_a):
        q, rows = O.dispatch_rows(idxs[s], pl[s][1], s, E_l, n_a, T)
        for t in range(T):
            for k in range(K):
                key = int(rows[t, k])
                assert key not in seen[q[t, k]]
                seen[q[t, k]].add(key)
                e_l = idxs[s][t, k] % E_l
                region = (e_l * n_a + s) * T
                assert region <= key < region + cnt[s, idxs[s][t, k]]
    for q in range(n_e):
        total, seg, base = layout[q]
        assert (seg % O.ROW_ALIGN == 0).all() and (np.diff(seg) >= total[:-1]).all()


def test_combine_matches_float64():
    T, K, H = 16, 4, 256
    y = O.synth_tokens(T * K, H, seed=3).reshape(T, K, H)
    w = np.random.default_rng(5).random((T, K), dtype=np.float32)
    r = O.synth_tokens(T, H, seed=6)
    out = O.combine(y, w, r)
    ref = O.bf16_to_f32(r).astype(np.float64) + np.einsum("tk,tkh->th", w.astype(np.float64),
                                                          O.bf16_to_f32(y).astype(np.float64))
    np.testing.assert_allclose(O.bf16_to_f32(out), ref, rtol=2 ** -7, atol=1e-6)


def test_expert_ffn_matches_float64():
    H, Hp, t = 256, 384, 20
    wts = O.synth_weights(H, Hp, 1, seed=7)
    x = O.synth_tokens(t, H, seed=8)
    y = O.expert_ffn(x, wts.w_gate[0], wts.w_up[0], wts.w_down[0])
    xf = O.bf16_to_f32(x).astype(np.float64)
    g = xf @ O.bf16_to_f32(wts.w_gate[0]).astype(np.float64).T
    u = xf @ O.bf16_to_f32(wts.w_up[0]).astype(np.float64).T
    h = g / (1 + np.exp(-g)) * u
    ref = h @ O.bf16_to_f32(wts.w_down[0]).astype(np.float64).T
    err = np.linalg.norm(O.bf16_to_f32(y) - ref) / np.linalg.norm(ref)
    assert err < 5e-3


# ---------------------------------------------------- golden fixtures -----
@pytest.mark.parametrize("name", ["tiny", "dbrx_router", "deepseek_router"])
def test_golden_fixtures(name):
    g = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    T, H, Hp, E, K = (int(v) for v in g["shape"])
    wts = O.synth_weights(H, Hp, E, seed=0, experts=None if name == "tiny" else [])
    x = O.synth_tokens(T, H, seed=1)
    assert hashlib.sha256(x.tobytes()).digest() == g["x_sha"].tobytes(), "input generator drifted"
    assert hashlib.sha256(wts.wg.tobytes()).digest() == g["wg_sha"].tobytes(), "weight generator drifted"
    idx, w, lg = O.router(x, wts.wg, K, want_logits=True)
    np.testing.assert_array_equal(lg.view(np.uint32), g["logits"].view(np.uint32))
    np.testing.assert_array_equal(idx, g["idx"])
    np.testing.assert_array_equal(w.view(np.uint32), g["w"].view(np.uint32))
    cnt, slot = O.place(idx, E)
    np.testing.assert_array_equal(cnt, g["cnt"])
    np.testing.assert_array_equal(slot, g["slot"])
    if name == "tiny":
        res = O.moe_layer([x], wts, K, n_e=1, resid=True)
        np.testing.assert_array_equal(res.y[0], g["y"])
        np.testing.assert_array_equal(res.out[0], g["out"])


def test_expert_tp_partials_sum_to_the_full_layer():
    """Expert TP (tp = 2 nodes of 2 GPUs): the per-rank partials y_r cover
    disjoint feature slices, their fp32 sum is the full expert output up to
    bf16 rounding, and the layer output matches tp = 1 within the bf16
    tolerance; routing / counts / placement are identical."""
    from _util import assert_close_bf16

    wts = O.synth_weights(512, 256, 8, seed=0)
    xs = [O.synth_tokens(24, 512, seed=11), O.synth_tokens(17, 512, seed=12)]
    r1 = O.moe_layer(xs, wts, 2, n_e=2)
    r2 = O.moe_layer(xs, wts, 2, n_e=4, tp=2)
    for s in range(2):
        np.testing.assert_array_equal(r1.idx[s], r2.idx[s])
        np.testing.assert_array_equal(r1.slot[s], r2.slot[s])
        assert r2.y[s].shape == (xs[s].shape[0], 2, 2, 512)
        ysum = O.bf16_to_f32(r2.y[s][:, :, 0]) + O.bf16_to_f32(r2.y[s][:, :, 1])
        assert_close_bf16(O.bf16_round(ysum), r1.y[s], "tp partial sum")
        assert_close_bf16(r2.out[s], r1.out[s], "tp layer output")
    np.testing.assert_array_equal(r1.cnt, r2.cnt)
    assert [len(l[0]) for l in r2.layout] == [4, 4]  # 2 nodes x E_l = 4


def test_decode_attention_c_matches_numpy():
    """The C attention used by the CPU baseline agrees with the readable numpy
    restatement (fp32 both; only the summation order differs)."""
    rng = np.random.default_rng(0)
    T, nh, nkv = 5, 12, 3
    lens = np.array([1, 64, 65, 200, 17], np.int32)
    need = (lens + 63) // 64
    bt = np.zeros((T, need.max()), np.int32)
    perm = rng.permutation(need.sum()).astype(np.int32)
    off = 0
    for t in range(T):
        bt[t, :need[t]] = perm[off:off + need[t]]
        off += need[t]
    kc = O.fill_normal((need.sum(), nkv, 64, 128), 1)
    vc = O.fill_normal((need.sum(), nkv, 64, 128), 2)
    q = O.fill_normal((T, nh, 128), 3, 0.2)
    a = O.bf16_to_f32(O.decode_attention(q, kc, vc, bt, lens)).astype(np.float64)
    b = O.bf16_to_f32(O.decode_attention_c(q, kc, vc, bt, lens)).astype(np.float64)
    assert np.abs(a - b).max() <= 2 ** -7 * np.abs(a).max()
    assert np.linalg.norm(a - b) / np.linalg.norm(a) < 1e-3


def test_fill_normal_thread_independent_and_normal():
    a = O.fill_normal((1 << 16,), 7, as_f32=True)
    b = O.bf16_to_f32(O.fill_normal((1 << 16,), 7))
    np.testing.assert_array_equal(a, b)
    assert abs(a.mean()) < 0.02 and abs(a.std() - 1.0) < 0.02


def test_cpu_decode_layer_matches_oracle_pieces():
    """The CPU baseline's layer step is the oracle's attention stage followed
    by the oracle's MoE layer (routing bit-exact, output within tolerance)."""
    H, Hp, E, K, T = 512, 256, 8, 2, 24
    ctx = np.random.default_rng(1).integers(1, 150, size=T).astype(np.int32)
    L = O.CpuDecodeLayer(H, Hp, E, K, T, n_heads=4, n_kv=2, ctx=ctx, seed=3)
    x = O.fill_normal((T, H), 9)
    kc, vc = L.k_cache.copy(), L.v_cache.copy()
    out, ph = L.step(x)
    assert ph["layer_s"] > 0
    wq = O.bf16_round(L.wqkv)
    wo = O.bf16_round(L.wo)
    h = O.attention_stage(x, wq, wo, ctx.copy(), 4, 2, L.theta, L.bt, kc, vc)
    wts = O.LayerWeights(L.wg, np.stack([O.bf16_round(w) for w in L.w_gate]),
                         np.stack([O.bf16_round(w) for w in L.w_up]), np.stack([O.bf16_round(w) for w in L.w_down]))
    ref = O.moe_layer([h], wts, K, n_e=1, resid=True)
    from _util import assert_close_bf16
    assert_close_bf16(out, ref.out[0], "cpu layer")
