"""GPU parity: every kernel against the CPU oracle on the same seeded inputs.

Bit-exact: router idx / counts / slots / weights, dispatch row placement,
combine (given identical expert outputs).  Tolerance (stated here):
expert FFN and layer outputs vs the oracle's fp32-accumulated reference with
the same bf16 rounding points -- rel-L2 <= 5e-3 and max-abs <= 2^-7 * max|ref|
(SURVEY.md §8c).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

from _util import assert_close_bf16  # noqa: E402


def to_dev(a_u16: np.ndarray) -> "torch.Tensor":
    return torch.from_numpy(a_u16.view(np.int16).copy()).view(torch.bfloat16).cuda()


def to_host(t) -> np.ndarray:
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


# ------------------------------------------------------------------ router --
ROUTER_CASES = [
    # T, H, E, K
    (64, 512, 8, 2),       # tiny config
    (1, 512, 8, 2),        # single token
    (37, 1024, 8, 2),      # ragged T
    (257, 4096, 8, 2),     # Mixtral-8x7B shape
    (130, 6144, 16, 4),    # DBRX shape
    (96, 7168, 256, 8),    # DeepSeek-V3 shape (E=256, BT=4 path)
    (2400, 7168, 256, 8),  # DeepSeek-V3 shape, BT=16 path
    (1024, 6144, 8, 2),    # Mixtral-8x22B shape at b_a = 1024
    (50, 512, 6, 3),       # E not a multiple of 4
]


@pytest.mark.parametrize("T,H,E,K", ROUTER_CASES)
def test_router_bit_exact(lib, T, H, E, K):
    from paper_2504_02263_b200 import ops

    x = O.synth_tokens(T, H, seed=1 + T)
    wg = O.synth_weights(H, 128, E, seed=0, experts=[]).wg
    idx_r, w_r = O.router(x, wg, K)
    cnt_r, slot_r = O.place(idx_r, E)
    idx, w, cnt, slot = ops.gate_topk(to_dev(x), to_dev(wg), K)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_r)
    np.testing.assert_array_equal(cnt.cpu().numpy(), cnt_r)
    np.testing.assert_array_equal(slot.cpu().numpy(), slot_r)
    # weights: bit-exact too (deterministic exp, IEEE division)
    np.testing.assert_array_equal(w.cpu().numpy().view(np.uint32), w_r.view(np.uint32))


def test_router_ties_prefer_lower_expert(lib):
    """All-equal logits: top-K must be experts 0..K-1 with equal weights."""
    from paper_2504_02263_b200 import ops

    T, H, E, K = 40, 512, 8, 3
    x = O.synth_tokens(T, H, seed=5)
    wg = np.zeros((E, H), np.uint16)  # all logits exactly 0
    idx, w, cnt, slot = ops.gate_topk(to_dev(x), to_dev(wg), K)
    idx_r, w_r = O.router(x, wg, K)
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_r)
    assert (idx_r == np.arange(K)).all()
    np.testing.assert_array_equal(w.cpu().numpy(), w_r)


def test_router_repeatable_workspace_reuse(lib):
    from paper_2504_02263_b200 import ops

    T, H, E, K = 300, 1024, 16, 4
    x = to_dev(O.synth_tokens(T, H, seed=9))
    wg = to_dev(O.synth_weights(H, 128, E, experts=[]).wg)
    ws = ops.RouterWorkspace(T, E)
    a = ops.gate_topk(x, wg, K, ws)
    outs = [t.clone() for t in a]
    for _ in range(3):
        b = ops.gate_topk(x, wg, K, ws)
        for u, v in zip(outs, b):
            assert torch.equal(u, v)


# ------------------------------------------------------------- grouped FFN --
FFN_CASES = [
    # H, Hp, totals per local expert
    (512, 1536, [20, 0, 77, 128, 129, 3, 64, 1]),
    (1024, 512, [300]),
    (4096, 1024, [130, 257]),
]


@pytest.mark.parametrize("H,Hp,totals", FFN_CASES)
def test_grouped_ffn_matches_oracle(lib, H, Hp, totals):
    from paper_2504_02263_b200 import ops

    E_l = len(totals)
    wts = O.synth_weights(H, Hp, E_l, seed=3)
    starts = ops.segment_starts(totals)
    rows = starts[-1] + (totals[-1] + 127) // 128 * 128 if totals else 0
    rows = max(rows, 128)
    x = np.zeros((rows, H), np.uint16)
    rng_x = O.synth_tokens(rows, H, seed=11)
    for s, t in zip(starts, totals):
        x[s:s + t] = rng_x[s:s + t]
    w13 = ops.pack_w13(to_dev(wts.w_gate), to_dev(wts.w_up))
    y = ops.grouped_ffn(to_dev(x), torch.tensor(totals, dtype=torch.int32), w13, to_dev(wts.w_down))
    torch.cuda.synchronize()
    y = to_host(y)
    for e, (s, t) in enumerate(zip(starts, totals)):
        if t == 0:
            continue
        ref = O.expert_ffn(x[s:s + t], wts.w_gate[e], wts.w_up[e], wts.w_down[e])
        assert_close_bf16(y[s:s + t], ref, f"expert {e}")


def test_pack_w13_layout(lib):
    from paper_2504_02263_b200 import ops

    E_l, Hp, H = 2, 256, 512
    g = torch.randn(E_l, Hp, H, device="cuda").to(torch.bfloat16)
    u = torch.randn(E_l, Hp, H, device="cuda").to(torch.bfloat16)
    w = ops.pack_w13(g, u)
    # every 256-row N tile: [gate 64 | up 64 | gate 64 | up 64] of 128 features
    ref = torch.stack([g.view(E_l, Hp // 64, 64, H), u.view(E_l, Hp // 64, 64, H)], dim=2).view(E_l, 2 * Hp, H)
    assert torch.equal(w, ref)


# ----------------------------------------------------------------- combine --
@pytest.mark.parametrize("T,K,H,resid", [(64, 2, 512, False), (33, 8, 7168, True), (1, 4, 6144, True)])
def test_combine_bit_exact(lib, T, K, H, resid):
    from paper_2504_02263_b200 import ops

    y = O.synth_tokens(T * K, H, seed=21).reshape(T, K, H)
    rng = np.random.default_rng(4)
    w = rng.random((T, K), dtype=np.float32)
    r = O.synth_tokens(T, H, seed=22) if resid else None
    out = ops.combine_local(to_dev(y), torch.from_numpy(w).cuda(), to_dev(r) if resid else None)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(to_host(out), O.combine(y, w, r))


# ------------------------------------------------- full layer, co-located --
def _colocated_layer(shape, b_a, m=1, seed=0):
    from paper_2504_02263_b200 import runtime
    from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec

    model = as_model_spec(shape)
    plan = DeploymentPlan(n_a=1, n_e=1, m=m, b_a=b_a, colocated=True)
    g = runtime.M2NGroup(model, plan, rank=0)
    wts = O.synth_weights(model.hidden, model.intermediate, model.experts, seed=seed)
    from paper_2504_02263_b200 import ops
    w13 = ops.pack_w13(to_dev(wts.w_gate), to_dev(wts.w_up))
    layer = runtime.MoEDecodeLayer(g, wg=to_dev(wts.wg), w13=w13, w2=to_dev(wts.w_down))
    return g, layer, wts, model


@pytest.mark.parametrize("T", [64, 17])
def test_colocated_layer_tiny(lib, T):
    g, layer, wts, model = _colocated_layer("tiny", b_a=64)
    x = O.synth_tokens(T, model.hidden, seed=1)
    xd = to_dev(x)
    r = layer.router(xd, 0)
    layer.dispatch(xd, r, 0)
    layer.expert_wait(0)
    torch.cuda.synchronize()
    recv = to_host(g.recv_view(0))  # rows as dispatched (the FFN then writes Y over them)
    layer.expert_ffn(0)
    out = layer.combine(r)
    torch.cuda.synchronize()
    assert g.status() == 0
    ref = O.moe_layer([x], wts, model.topk, n_e=1)
    # bit-exact routing and placement
    np.testing.assert_array_equal(r.idx[:T].cpu().numpy(), ref.idx[0])
    np.testing.assert_array_equal(r.cnt.cpu().numpy(), ref.cnt[0])
    np.testing.assert_array_equal(r.slot[:T].cpu().numpy(), ref.slot[0])
    q, rows = O.dispatch_rows(ref.idx[0], ref.slot[0], 0, model.experts, 1, g.plan.b_a)
    t_idx, k_idx = np.nonzero(np.ones_like(ref.idx[0], bool))
    np.testing.assert_array_equal(recv[rows[t_idx, k_idx]], x[t_idx])
    # expert outputs (tolerance), then combine bit-exact given the GPU's own y
    ybuf = to_host(layer.gather_y(r))
    assert_close_bf16(ybuf, ref.y[0], "expert outputs")
    np.testing.assert_array_equal(to_host(out), O.combine(ybuf, r.w[:T].cpu().numpy()))
    assert_close_bf16(to_host(out), ref.out[0], "layer output")
    g.close()


def test_colocated_layer_epochs_and_slots(lib):
    """Several micro-batch slots reused over several layers: epochs advance,
    buffers are reused, results stay exact for each (mb, layer)."""
    g, layer, wts, model = _colocated_layer("tiny", b_a=48, m=3)
    for l in range(3):
        for j in range(3):
            x = O.synth_tokens(48 - 5 * j, model.hidden, seed=100 + 10 * l + j)
            xd = to_dev(x)
            r = layer.router(xd, j)
            layer.dispatch(xd, r, j)
            layer.expert_step(j)
            out = layer.combine(r, resid=xd)
            torch.cuda.synchronize()
            ref = O.moe_layer([x], wts, model.topk, n_e=1, resid=True)
            np.testing.assert_array_equal(r.idx[:r.T].cpu().numpy(), ref.idx[0])
            assert_close_bf16(to_host(out), ref.out[0], f"layer {l} mb {j}")
    assert g.status() == 0
    g.close()


def test_colocated_layer_mixtral_shape(lib):
    """Mixtral-8x22B-shaped layer (h=6144, h'=16384, E=8, K=2) at b_a=256:
    routing/placement bit-exact, outputs within tolerance (oracle on a subset of
    experts to bound CPU time)."""
    g, layer, wts, model = _colocated_layer("mixtral-8x22b", b_a=256)
    T = 256
    x = O.synth_tokens(T, model.hidden, seed=7)
    xd = to_dev(x)
    r = layer.router(xd, 0)
    layer.dispatch(xd, r, 0)
    layer.expert_step(0)
    out = layer.combine(r)
    torch.cuda.synchronize()
    assert g.status() == 0
    idx_r, w_r = O.router(x, wts.wg, model.topk)
    cnt_r, slot_r = O.place(idx_r, model.experts)
    np.testing.assert_array_equal(r.idx.cpu().numpy(), idx_r)
    np.testing.assert_array_equal(r.slot.cpu().numpy(), slot_r)
    ybuf = to_host(layer.gather_y(r))
    for e in (0, 5):
        t, k = np.nonzero(idx_r == e)
        order = np.argsort(slot_r[t, k])
        t, k = t[order], k[order]
        ref = O.expert_ffn(x[t], wts.w_gate[e], wts.w_up[e], wts.w_down[e])
        assert_close_bf16(ybuf[t, k], ref, f"expert {e}")
    np.testing.assert_array_equal(to_host(out), O.combine(ybuf, w_r))
    g.close()


def test_pingpong_runner_colocated(lib):
    """PingPongRunner over L layers with m slots equals the layer-by-layer
    oracle on the GPU's own per-layer routing (routing bit-exact each layer)."""
    from paper_2504_02263_b200 import runtime

    g, layer, wts, model = _colocated_layer("tiny", b_a=32, m=2)
    xs0 = [O.synth_tokens(32, model.hidden, seed=50 + j) for j in range(2)]
    xs = [to_dev(x) for x in xs0]
    run = runtime.PingPongRunner(layer, layers=3)
    run.run(xs)
    torch.cuda.synchronize()
    assert g.status() == 0
    for j in range(2):
        cur = xs0[j]
        for _ in range(3):
            cur = O.moe_layer([cur], wts, model.topk, n_e=1, resid=True).out[0]
        assert_close_bf16(to_host(xs[j]), cur, f"mb {j} after 3 layers")
    g.close()


def test_echo_round_trip_bit_exact(lib):
    """dispatch -> identity expert -> combine returns every row to its (t, k)
    slot: out = combine(y = x per k) exactly (pure M2N path)."""
    from paper_2504_02263_b200 import runtime
    from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec

    model = as_model_spec("dbrx")
    g = runtime.M2NGroup(model, DeploymentPlan(n_a=1, n_e=1, m=2, b_a=40, colocated=True), rank=0)
    wg = O.synth_weights(model.hidden, 128, model.experts, experts=[]).wg
    layer = runtime.MoEDecodeLayer(g, wg=to_dev(wg))
    for j, T in enumerate((40, 13)):
        x = O.synth_tokens(T, model.hidden, seed=30 + j)
        xd = to_dev(x)
        r = layer.router(xd, j)
        layer.dispatch(xd, r, j)
        layer.expert_echo(j)
        out = layer.combine(r)
        torch.cuda.synchronize()
        y = np.repeat(x[:, None, :], model.topk, axis=1)
        np.testing.assert_array_equal(to_host(layer.gather_y(r)), y)
        np.testing.assert_array_equal(to_host(out), O.combine(y, r.w[:T].cpu().numpy()))
    assert g.status() == 0
    g.close()


def test_graph_replay_device_epochs(lib):
    """A captured step replays with device-tracked epochs: every replay is the
    next use of each slot, results equal the eager (explicit-epoch) run."""
    from paper_2504_02263_b200 import runtime

    g, layer, wts, model = _colocated_layer("tiny", b_a=32, m=2)
    xs0 = [O.synth_tokens(32, model.hidden, seed=70 + j) for j in range(2)]
    xs = [to_dev(x) for x in xs0]
    run = runtime.PingPongRunner(layer, layers=2, chain=False)
    run.run(xs)                      # eager, explicit epochs
    torch.cuda.synchronize()
    eager = [to_host(o) for o in run.outs]
    run.capture(xs)                  # switches to device epochs
    for _ in range(3):
        run.replay()
    torch.cuda.synchronize()
    assert g.status() == 0
    for j in range(2):
        np.testing.assert_array_equal(to_host(run.outs[j]), eager[j])
        ref = O.moe_layer([xs0[j]], wts, model.topk, n_e=1, resid=True).out[0]
        assert_close_bf16(to_host(run.outs[j]), ref, f"mb {j}")
    g.close()


def test_stale_explicit_epoch_is_rejected(lib):
    """An explicit epoch that disagrees with the device's use count must not
    race (the arrival counters are cumulative): the dispatch refuses, sets
    MSI_ESTATE, and sends nothing."""
    from paper_2504_02263_b200 import runtime
    from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec

    model = as_model_spec("tiny")
    g = runtime.M2NGroup(model, DeploymentPlan(n_a=1, n_e=1, m=1, b_a=16, colocated=True), rank=0,
                         timeout_s=0.5)
    layer = runtime.MoEDecodeLayer(g, wg=to_dev(O.synth_weights(model.hidden, 128, 8, experts=[]).wg))
    x = to_dev(O.synth_tokens(16, model.hidden, seed=3))
    r = layer.router(x, 0)
    layer.dispatch(x, r, 0)            # device epoch 1
    layer.expert_echo(0)
    layer.combine(r)
    torch.cuda.synchronize()
    assert g.status() == 0
    layer.device_epochs = False         # host count says 1 again: stale
    layer.epoch_a[0] = 0
    r = layer.router(x, 0)
    layer.dispatch(x, r, 0)
    torch.cuda.synchronize()
    assert g.status() == -3             # MSI_ESTATE
    g.close()


def test_colocated_layer_256_experts(lib):
    """Fine-grained routing (E=256, top-8) with all 256 experts on one GPU:
    exercises the large segment-table GEMM variant and the E=256 router."""
    shape = {"name": "fine256", "layers": 1, "hidden": 512, "intermediate": 256, "experts": 256, "topk": 8}
    g, layer, wts, model = _colocated_layer(shape, b_a=96)
    x = O.synth_tokens(96, model.hidden, seed=12)
    xd = to_dev(x)
    r = layer.router(xd, 0)
    layer.dispatch(xd, r, 0)
    layer.expert_step(0)
    out = layer.combine(r, resid=xd)
    torch.cuda.synchronize()
    assert g.status() == 0
    ref = O.moe_layer([x], wts, model.topk, n_e=1, resid=True)
    np.testing.assert_array_equal(r.idx.cpu().numpy(), ref.idx[0])
    np.testing.assert_array_equal(r.slot.cpu().numpy(), ref.slot[0])
    assert_close_bf16(to_host(layer.gather_y(r)), ref.y[0], "expert outputs")
    assert_close_bf16(to_host(out), ref.out[0], "layer output")
    g.close()


def _replicated_slots():
    """Tiny model, one expert GPU, experts 0-3 replicated: 12 physical slots."""
    from paper_2504_02263_b200.balance import SlotPlacement
    phys2log = np.array([0, 1, 2, 3, 4, 5, 6, 7, 0, 1, 2, 3], np.int32)
    rep = np.zeros((8, 3), np.int32)
    for e in range(8):
        ps = np.flatnonzero(phys2log == e)
        rep[e, 0] = len(ps)
        rep[e, 1:1 + len(ps)] = ps
    return SlotPlacement(8, 1, 12, phys2log, rep, 2)


def test_replicated_experts_bit_identical(lib):
    """Routing to replicated expert slots (load balancing) changes placement but
    not results: pidx / counts / slots bit-exact vs the oracle, layer output
    bit-identical to the unreplicated GPU run."""
    from paper_2504_02263_b200 import ops, runtime
    from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec

    model = as_model_spec("tiny")
    wts = O.synth_weights(model.hidden, model.intermediate, model.experts, seed=0)
    x = O.synth_tokens(64, model.hidden, seed=41)
    outs = {}
    for name, sl in (("plain", None), ("rep", _replicated_slots())):
        g = runtime.M2NGroup(model, DeploymentPlan(n_a=1, n_e=1, m=1, b_a=64, colocated=True), rank=0, slots=sl)
        ex = runtime.local_experts(g)
        w13 = ops.pack_w13(to_dev(wts.w_gate[ex]), to_dev(wts.w_up[ex]))
        layer = runtime.MoEDecodeLayer(g, wg=to_dev(wts.wg), w13=w13, w2=to_dev(wts.w_down[ex]))
        xd = to_dev(x)
        r = layer.router(xd, 0)
        layer.dispatch(xd, r, 0)
        layer.expert_step(0)
        out = layer.combine(r, resid=xd)
        torch.cuda.synchronize()
        assert g.status() == 0
        outs[name] = to_host(out)
        if sl is not None:
            ref = O.moe_layer([x], wts, model.topk, n_e=1, resid=True, rep=sl.rep, phys2log=sl.phys2log)
            np.testing.assert_array_equal(r.idx.cpu().numpy(), ref.idx[0])
            np.testing.assert_array_equal(r.pidx.cpu().numpy(), ref.pidx[0])
            np.testing.assert_array_equal(r.cnt.cpu().numpy(), ref.cnt[0])
            np.testing.assert_array_equal(r.slot.cpu().numpy(), ref.slot[0])
            assert (r.cnt.cpu().numpy()[8:] > 0).all()  # the replicas received tokens
        g.close()
    np.testing.assert_array_equal(outs["rep"], outs["plain"])


@pytest.mark.parametrize("tile,T,H,E,K", [("2x16x4", 130, 7168, 256, 8), ("8x8x32", 2400, 7168, 256, 8),
                                          ("4x4x16", 333, 4096, 64, 6), ("2x16x16", 1024, 6144, 16, 4),
                                          ("1x8x8", 77, 6144, 8, 2)])
def test_router_tile_variants_bit_exact(lib, monkeypatch, tile, T, H, E, K):
    """Every logit kernel variant (MSI_ROUTER_TILE) keeps the pinned reduction
    order: routing, counts, slots and weights bit-identical to the oracle."""
    from paper_2504_02263_b200 import ops

    monkeypatch.setenv("MSI_ROUTER_TILE", tile)
    x = O.synth_tokens(T, H, seed=5 + T)
    wg = O.synth_weights(H, 128, E, seed=3, experts=[]).wg
    idx_r, w_r = O.router(x, wg, K)
    cnt_r, slot_r = O.place(idx_r, E)
    idx, w, cnt, slot = ops.gate_topk(to_dev(x), to_dev(wg), K)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_r)
    np.testing.assert_array_equal(cnt.cpu().numpy(), cnt_r)
    np.testing.assert_array_equal(slot.cpu().numpy(), slot_r)
    np.testing.assert_array_equal(w.cpu().numpy().view(np.uint32), w_r.view(np.uint32))


@pytest.mark.parametrize("split,T,H,E,K", [("default", 130, 7168, 256, 8), ("default", 2400, 7168, 256, 8),
                                           ("4x32x64", 777, 7168, 256, 8), ("2x4x32", 301, 7168, 256, 8),
                                           ("1x1x128", 40, 7168, 256, 8), ("4x8x64", 515, 4096, 64, 6),
                                           ("0", 515, 4096, 64, 6)])
def test_router_split_path_bit_exact(lib, monkeypatch, split, T, H, E, K):
    """Fine-grained MoE (E >= 64): the logits kernel on its (token x expert) grid
    plus the route kernel give routing, counts, slots and weights bit-identical
    to the oracle for every tile choice (MSI_ROUTER_SPLIT; 0 = fused kernel)."""
    from paper_2504_02263_b200 import ops

    if split != "default":
        monkeypatch.setenv("MSI_ROUTER_SPLIT", split)
    x = O.synth_tokens(T, H, seed=9 + T)
    wg = O.synth_weights(H, 128, E, seed=4, experts=[]).wg
    idx_r, w_r = O.router(x, wg, K)
    cnt_r, slot_r = O.place(idx_r, E)
    idx, w, cnt, slot = ops.gate_topk(to_dev(x), to_dev(wg), K)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_r)
    np.testing.assert_array_equal(cnt.cpu().numpy(), cnt_r)
    np.testing.assert_array_equal(slot.cpu().numpy(), slot_r)
    np.testing.assert_array_equal(w.cpu().numpy().view(np.uint32), w_r.view(np.uint32))


# ------------------------------------------------------------- edge cases --
def test_router_nonfinite_tokens_bit_exact(lib):
    """Rows with NaN / +-Inf entries: NaN logits rank as -inf, ties go to the
    lower expert; idx / counts / slots / weights still bit-exact vs the oracle."""
    from paper_2504_02263_b200 import ops

    T, H, E, K = 40, 512, 8, 2
    x = O.synth_tokens(T, H, seed=31)
    x[3, 7] = 0x7FC0          # NaN -> every logit of token 3 is NaN
    x[5, :] = 0x7F80          # +Inf row -> +-Inf / NaN logits
    x[9, 100] = 0xFF80        # one -Inf entry
    wg = O.synth_weights(H, 128, E, seed=0, experts=[]).wg
    idx_r, w_r = O.router(x, wg, K)
    cnt_r, slot_r = O.place(idx_r, E)
    idx, w, cnt, slot = ops.gate_topk(to_dev(x), to_dev(wg), K)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_r)
    np.testing.assert_array_equal(cnt.cpu().numpy(), cnt_r)
    np.testing.assert_array_equal(slot.cpu().numpy(), slot_r)
    # weights: bit-exact where finite; NaN exactly where the oracle's softmax is
    # NaN (NaN payload bits differ between x86 and CUDA, so compare the class)
    wg_ = w.cpu().numpy()
    fin = np.isfinite(w_r)
    np.testing.assert_array_equal(np.isnan(wg_), np.isnan(w_r))
    np.testing.assert_array_equal(wg_[fin].view(np.uint32), w_r[fin].view(np.uint32))
    assert fin[[0, 1, 2, 4]].all()


def test_colocated_layer_concentrated_routing(lib):
    """Every token routed to the same two experts (a collision-heavy load):
    six experts get empty segments, two get all T rows; placement bit-exact,
    outputs within tolerance."""
    from paper_2504_02263_b200 import ops, runtime
    from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec

    model = as_model_spec("tiny")
    T = 96
    plan = DeploymentPlan(n_a=1, n_e=1, m=1, b_a=T, colocated=True)
    g = runtime.M2NGroup(model, plan, rank=0)
    wts = O.synth_weights(model.hidden, model.intermediate, model.experts, seed=0)
    x = O.synth_tokens(T, model.hidden, seed=41)
    # a shared constant feature that only experts 3 and 6 respond to (logit
    # shifts +32 / +24 against N(0, 1) logits): top-2 = {3, 6} for every token
    x[:, 0] = O.bf16_round(np.full(T, 8.0, np.float32))
    wgf = O.bf16_to_f32(wts.wg).copy()
    wgf[:, 0] = 0.0
    wgf[3, 0], wgf[6, 0] = 4.0, 3.0
    wts.wg[:] = O.bf16_round(wgf)
    w13 = ops.pack_w13(to_dev(wts.w_gate), to_dev(wts.w_up))
    layer = runtime.MoEDecodeLayer(g, wg=to_dev(wts.wg), w13=w13, w2=to_dev(wts.w_down))
    xd = to_dev(x)
    r = layer.router(xd, 0)
    layer.dispatch(xd, r, 0)
    layer.expert_step(0)
    out = layer.combine(r)
    torch.cuda.synchronize()
    assert g.status() == 0
    ref = O.moe_layer([x], wts, model.topk, n_e=1)
    assert set(np.unique(ref.idx[0])) == {3, 6}, "construction should route every token to experts 3 and 6"
    np.testing.assert_array_equal(r.idx[:T].cpu().numpy(), ref.idx[0])
    np.testing.assert_array_equal(r.cnt.cpu().numpy(), ref.cnt[0])
    np.testing.assert_array_equal(r.slot[:T].cpu().numpy(), ref.slot[0])
    ybuf = to_host(layer.gather_y(r))
    assert_close_bf16(ybuf, ref.y[0], "expert outputs")
    np.testing.assert_array_equal(to_host(out), O.combine(ybuf, r.w[:T].cpu().numpy()))
    g.close()


def test_colocated_layer_empty_microbatch(lib):
    """A micro-batch with T = 0 tokens still runs the whole protocol (counts,
    arrival and combine signals advance) and the next micro-batch is exact."""
    g, layer, wts, model = _colocated_layer("tiny", b_a=32)
    for T in (0, 32, 0, 5):
        x = O.synth_tokens(max(T, 1), model.hidden, seed=50 + T)[:T]
        xd = to_dev(x) if T else torch.empty((0, model.hidden), dtype=torch.bfloat16, device="cuda")
        r = layer.router(xd, 0)
        layer.dispatch(xd, r, 0)
        layer.expert_step(0)
        out = layer.combine(r)
        torch.cuda.synchronize()
        assert g.status() == 0, f"device status after T={T}"
        assert out.shape == (T, model.hidden)
        if T:
            ref = O.moe_layer([x], wts, model.topk, n_e=1)
            np.testing.assert_array_equal(r.idx[:T].cpu().numpy(), ref.idx[0])
            assert_close_bf16(to_host(out), ref.out[0], f"layer output T={T}")
        else:
            assert int(r.cnt.sum()) == 0
    g.close()


# ------------------------------------------- fused router + M2N dispatch --
@pytest.mark.parametrize("shape,T,b_a", [("tiny", 64, 64), ("tiny", 1, 64), ("dbrx", 333, 400),
                                         ("mixtral-8x22b", 3072, 3072),
                                         ({"name": "fine256", "layers": 1, "hidden": 7168, "intermediate": 256,
                                           "experts": 256, "topk": 8}, 700, 700),
                                         ({"name": "fine256s", "layers": 1, "hidden": 7168, "intermediate": 256,
                                           "experts": 256, "topk": 8}, 130, 130)])
def test_route_dispatch_fused_matches_oracle(lib, shape, T, b_a):
    """msi_route_dispatch (router + dispatch in one launch, decoupled
    look-back slots) places every row where the oracle says, with the same
    idx / w / cnt / slot bit-exact, and the echo round trip returns them."""
    from paper_2504_02263_b200 import runtime
    from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec

    model = as_model_spec(shape)
    g = runtime.M2NGroup(model, DeploymentPlan(n_a=1, n_e=1, m=2, b_a=b_a, colocated=True), rank=0)
    wg = O.synth_weights(model.hidden, 128, model.experts, seed=2, experts=[]).wg
    layer = runtime.MoEDecodeLayer(g, wg=to_dev(wg))
    for j, seed in enumerate((5, 6)):
        x = O.synth_tokens(T, model.hidden, seed=seed)
        xd = to_dev(x)
        r = layer.route_dispatch(xd, j)
        layer.expert_echo(j)
        out = layer.combine(r)
        torch.cuda.synchronize()
        assert g.status() == 0
        idx_r, w_r = O.router(x, wg, model.topk)
        cnt_r, slot_r = O.place(idx_r, model.experts)
        np.testing.assert_array_equal(r.idx[:T].cpu().numpy(), idx_r)
        np.testing.assert_array_equal(r.w[:T].cpu().numpy().view(np.uint32), w_r.view(np.uint32))
        np.testing.assert_array_equal(r.cnt.cpu().numpy(), cnt_r)
        np.testing.assert_array_equal(r.slot[:T].cpu().numpy(), slot_r)
        _, rows = O.dispatch_rows(idx_r, slot_r, 0, model.experts, 1, b_a)
        recv = to_host(g.recv_view(j))  # the identity expert leaves the rows in place
        for k in range(model.topk):
            np.testing.assert_array_equal(recv[rows[:, k]], x)
        y = np.repeat(x[:, None, :], model.topk, axis=1)
        np.testing.assert_array_equal(to_host(out), O.combine(y, w_r))
    g.close()


def test_route_dispatch_fused_empty_and_replicated(lib):
    """T = 0 still runs the protocol (zero counts, release); replicated slots
    route through the fused kernel bit-exactly and give the same output as the
    unreplicated layer."""
    from paper_2504_02263_b200 import ops, runtime
    from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec

    model = as_model_spec("tiny")
    wts = O.synth_weights(model.hidden, model.intermediate, model.experts, seed=0)
    x = O.synth_tokens(64, model.hidden, seed=41)
    outs = {}
    for name, sl in (("plain", None), ("rep", _replicated_slots())):
        g = runtime.M2NGroup(model, DeploymentPlan(n_a=1, n_e=1, m=1, b_a=64, colocated=True), rank=0, slots=sl)
        ex = runtime.local_experts(g)
        w13 = ops.pack_w13(to_dev(wts.w_gate[ex]), to_dev(wts.w_up[ex]))
        layer = runtime.MoEDecodeLayer(g, wg=to_dev(wts.wg), w13=w13, w2=to_dev(wts.w_down[ex]))
        empty = torch.empty((0, model.hidden), dtype=torch.bfloat16, device="cuda")
        r = layer.route_dispatch(empty, 0)
        layer.expert_step(0)
        layer.combine(r)
        torch.cuda.synchronize()
        assert g.status() == 0 and int(r.cnt.sum()) == 0
        xd = to_dev(x)
        r = layer.route_dispatch(xd, 0)
        layer.expert_step(0)
        out = layer.combine(r, resid=xd)
        torch.cuda.synchronize()
        assert g.status() == 0
        outs[name] = to_host(out)
        ref = O.moe_layer([x], wts, model.topk, n_e=1, resid=True,
                          rep=None if sl is None else sl.rep, phys2log=None if sl is None else sl.phys2log)
        np.testing.assert_array_equal(r.idx.cpu().numpy(), ref.idx[0])
        np.testing.assert_array_equal(r.dest.cpu().numpy(), ref.pidx[0])
        np.testing.assert_array_equal(r.cnt.cpu().numpy(), ref.cnt[0])
        np.testing.assert_array_equal(r.slot.cpu().numpy(), ref.slot[0])
        assert_close_bf16(outs[name], ref.out[0], f"layer output ({name})")
        g.close()
    np.testing.assert_array_equal(outs["rep"], outs["plain"])


@pytest.mark.parametrize("n_src,E_l,per", [(1, 3, 300), (2, 4, 200), (3, 2, 130), (8, 2, 70), (5, 5, 40)])
def test_expert_ffn_regions_equal_compact(lib, n_src, E_l, per):
    """The receive-region layout msi_expert_ffn reads (n_src regions per
    expert, A loaded as region runs; ragged, empty and one-row regions) gives
    bit-identical expert outputs to the same rows packed compactly per
    expert: every row's MMAs and epilogue are the same."""
    import torch

    from paper_2504_02263_b200 import ops, runtime
    from paper_2504_02263_b200.config import MoeModelSpec

    model = MoeModelSpec("regions", 1, 512, 768, E_l, 1)
    rng = np.random.default_rng(n_src * 31 + E_l)
    counts = rng.integers(0, 2 * per, size=(n_src, E_l))
    counts[0, 0] = 0
    if n_src > 1:
        counts[1, 0] = 1
    cap = int(counts.max()) + 5
    _, w13, w2 = runtime.synth_device_weights(model, list(range(E_l)), seed=3, device="cuda")
    x_reg = torch.randn((E_l * n_src * cap, model.hidden), device="cuda").to(torch.bfloat16)
    tot = counts.sum(0)
    starts = ops.segment_starts(tot.tolist())
    rows = starts[-1] + (int(tot[-1]) + 127) // 128 * 128 + 128
    xc = torch.zeros((rows, model.hidden), dtype=torch.bfloat16, device="cuda")
    for e in range(E_l):
        o = starts[e]
        for s in range(n_src):
            b = (e * n_src + s) * cap
            xc[o:o + counts[s, e]] = x_reg[b:b + counts[s, e]]
            o += counts[s, e]
    yc = ops.grouped_ffn(xc, torch.tensor(tot, dtype=torch.int32), w13, w2)
    y_reg = ops.grouped_ffn_regions(x_reg, counts, cap, w13, w2)
    xr = x_reg.clone()
    y_inplace = ops.grouped_ffn_regions(xr, counts, cap, w13, w2, y_reg=xr)  # Y over X
    y_gather = ops.grouped_ffn_regions(x_reg, counts, cap, w13, w2, gather=True)  # gathered, compact GEMM1
    torch.cuda.synchronize()
    for e in range(E_l):
        o = starts[e]
        for s in range(n_src):
            b = (e * n_src + s) * cap
            assert torch.equal(y_reg[b:b + counts[s, e]], yc[o:o + counts[s, e]]), (e, s)
            assert torch.equal(y_inplace[b:b + counts[s, e]], yc[o:o + counts[s, e]]), (e, s)
            assert torch.equal(y_gather[b:b + counts[s, e]], yc[o:o + counts[s, e]]), (e, s)
            o += counts[s, e]


@pytest.mark.parametrize("T,H,E,K,mode", [(130, 7168, 256, 8, "rand"), (2400, 7168, 256, 8, "rand"),
                                          (4096, 7168, 256, 8, "rand"), (515, 4096, 512, 8, "rand"),
                                          (300, 7168, 256, 8, "ties"), (64, 7168, 256, 8, "nonfinite")])
def test_router_tensor_core_path_bit_exact(lib, monkeypatch, T, H, E, K, mode):
    """Fine-grained router with the logits on tcgen05 (MSI_ROUTER_TC=1): the
    candidate experts of every token (within the fp32 error bound of the
    K-th) are recomputed in the pinned order, so idx / weights / counts /
    slots stay bit-exact vs the oracle -- including exact ties (duplicated
    gate rows: ties go to the lower expert) and non-finite rows (all experts
    recomputed)."""
    from paper_2504_02263_b200 import ops

    monkeypatch.setenv("MSI_ROUTER_TC", "1")
    x = O.synth_tokens(T, H, seed=11 + T)
    wg = O.synth_weights(H, 128, E, seed=6, experts=[]).wg
    if mode == "ties":  # experts 2k and 2k+1 identical: every logit ties with a neighbour
        wg = wg.copy()
        wg[1::2] = wg[0::2]
    if mode == "nonfinite":
        x = x.copy()
        x[3, 7] = 0x7FC0
        x[5, :] = 0x7F80
        x[9, 100] = 0xFF80
    idx_r, w_r = O.router(x, wg, K)
    cnt_r, slot_r = O.place(idx_r, E)
    idx, w, cnt, slot = ops.gate_topk(to_dev(x), to_dev(wg), K)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(idx.cpu().numpy(), idx_r)
    np.testing.assert_array_equal(cnt.cpu().numpy(), cnt_r)
    np.testing.assert_array_equal(slot.cpu().numpy(), slot_r)
    wgot = w.cpu().numpy()
    fin = np.isfinite(w_r)
    np.testing.assert_array_equal(np.isnan(wgot), np.isnan(w_r))
    np.testing.assert_array_equal(wgot[fin].view(np.uint32), w_r[fin].view(np.uint32))


@pytest.mark.timeout(300)
@pytest.mark.parametrize("rank", [0, 1, 2, 3])
def test_expert_ffn_many_experts_many_senders_regression(lib, rank):
    """Regression: 64 local experts x 4 senders (DeepSeek-V3 shape, co-located
    4 GPUs, 2048 tokens per rank -- counts captured from that run,
    tests/golden/hang/).  More than 32 (sender, expert) totals are summed by
    several warps; the segment table must wait for all of them, or the two
    CTAs of a pair disagree on the tile list and hang.  Every repetition must
    finish and give bit-identical rows to the compact layout."""
    import os

    import torch

    from paper_2504_02263_b200 import ops, runtime
    from paper_2504_02263_b200.config import MoeModelSpec

    here = os.path.dirname(os.path.abspath(__file__))
    counts = np.load(os.path.join(here, "golden", "hang", f"dbg_counts_r{rank}.npy"))
    n_src, E_l = counts.shape
    cap = int(counts.max()) + 3
    model = MoeModelSpec("hang", 1, 512, 256, E_l, 1)
    _, w13, w2 = runtime.synth_device_weights(model, list(range(E_l)), seed=1, device="cuda")
    x_reg = torch.randn((E_l * n_src * cap, model.hidden), device="cuda").to(torch.bfloat16)
    tot = counts.sum(0)
    starts = ops.segment_starts(tot.tolist())
    rows = starts[-1] + (int(tot[-1]) + 127) // 128 * 128 + 128
    xc = torch.zeros((rows, model.hidden), dtype=torch.bfloat16, device="cuda")
    for e in range(E_l):
        o = starts[e]
        for s in range(n_src):
            b = (e * n_src + s) * cap
            xc[o:o + counts[s, e]] = x_reg[b:b + counts[s, e]]
            o += counts[s, e]
    yc = ops.grouped_ffn(xc, torch.tensor(tot, dtype=torch.int32), w13, w2)
    for rep in range(4):
        for gather in (True, False):
            y = ops.grouped_ffn_regions(x_reg, counts, cap, w13, w2, gather=gather)
            torch.cuda.synchronize()
            for e in range(0, E_l, 7):
                o = starts[e]
                for s in range(n_src):
                    b = (e * n_src + s) * cap
                    assert torch.equal(y[b:b + counts[s, e]], yc[o:o + counts[s, e]]), (rep, gather, e, s)
                    o += counts[s, e]
