"""GPU parity at the shapes the bench runs.

* The bench's N = 1 configuration exactly: Mixtral-8x22B-shaped layer
  (h 6144, h' 16384, E 8, K 2), co-located, m = 3 micro-batches of b_a = 1024
  merged into T = 3072 tokens, weights from runtime.synth_device_weights (the
  bench's generator): routing (idx, w, cnt, slot) and receive-row placement
  bit-exact over all 3072 tokens; every expert's outputs (t_e ~ 768: full CTA
  -pair tiles over h' = 16384, several scheduler waves) within the bf16
  tolerance of the oracle; combine bit-exact given the GPU's expert outputs;
  layer output within tolerance.
* The grouped SwiGLU GEMM at the other BASELINE shapes:
  DBRX (h 6144, h' 10752, 4 local experts), Mixtral-8x7B (h 4096, h' 14336,
  2 local experts), DeepSeek-V3-shaped (h 7168, h' 2048, 64 local experts,
  ragged loads incl. empty and odd-tile segments), sampled experts vs the
  oracle.

Tolerance: rel-L2 <= 5e-3 and max-abs <= 2^-7 max|ref| (tests/_util.py).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

from _util import assert_close_bf16  # noqa: E402


def to_host(t) -> np.ndarray:
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def unpack_w13(w13_e: "torch.Tensor"):
    """Inverse of msi_pack_w13 for one expert: [2H', H] -> gate, up [H', H]
    (every 256 rows = [gate 64 | up 64 | gate 64 | up 64] of 128 features)."""
    two_hp, H = w13_e.shape
    v = w13_e.view(two_hp // 256, 2, 2, 64, H)  # [j, half, gate/up, i, H]
    gate = v[:, :, 0].reshape(two_hp // 2, H)
    up = v[:, :, 1].reshape(two_hp // 2, H)
    return gate, up


def test_unpack_w13_inverts_pack(lib):
    from paper_2504_02263_b200 import ops

    g = torch.randn(2, 256, 512, device="cuda").to(torch.bfloat16)
    u = torch.randn(2, 256, 512, device="cuda").to(torch.bfloat16)
    w = ops.pack_w13(g, u)
    for e in range(2):
        gg, uu = unpack_w13(w[e])
        assert torch.equal(gg, g[e]) and torch.equal(uu, u[e])


def test_bench_config_n1_mixtral_8x22b(lib):
    """The exact layer bench.py times at N = 1 (co-located, T = 3072)."""
    from paper_2504_02263_b200 import runtime
    from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec

    model = as_model_spec("mixtral-8x22b")
    T = 3 * 1024
    plan = DeploymentPlan(n_a=1, n_e=1, m=1, b_a=T, colocated=True)
    g = runtime.M2NGroup(model, plan, rank=0)
    dev = g.device
    wg, w13, w2 = runtime.synth_device_weights(model, runtime.local_experts(g), seed=0, device=dev)
    layer = runtime.MoEDecodeLayer(g, wg=wg, w13=w13, w2=w2)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)  # bench.py: rank 0's token generator
    xd = torch.randn((T, model.hidden), generator=gen, device=dev).to(torch.bfloat16)
    r = layer.router(xd, 0)
    layer.dispatch(xd, r, 0)
    layer.expert_wait(0)
    torch.cuda.synchronize()
    recv = to_host(g.recv_view(0))  # rows as dispatched (the FFN then writes Y over them)
    layer.expert_ffn(0)
    out = layer.combine(r, resid=xd)
    torch.cuda.synchronize()
    assert g.status() == 0
    x = to_host(xd)
    wg_h = to_host(wg)
    idx_r, w_r = O.router(x, wg_h, model.topk)
    cnt_r, slot_r = O.place(idx_r, model.experts)
    np.testing.assert_array_equal(r.idx.cpu().numpy(), idx_r)
    np.testing.assert_array_equal(r.w.cpu().numpy().view(np.uint32), w_r.view(np.uint32))
    np.testing.assert_array_equal(r.cnt.cpu().numpy(), cnt_r)
    np.testing.assert_array_equal(r.slot.cpu().numpy(), slot_r)
    assert cnt_r.min() >= 512, "every expert should see a full multi-tile segment at this shape"
    # placement: every (t, k) row at the oracle's receive row
    _, rows = O.dispatch_rows(idx_r, slot_r, 0, model.experts, 1, T)
    np.testing.assert_array_equal(recv[rows[:, 0]], x)
    np.testing.assert_array_equal(recv[rows[:, 1]], x)
    # every expert's SwiGLU outputs (t_e ~ 768) vs the oracle
    ybuf = to_host(layer.gather_y(r))
    y_ref = np.zeros_like(ybuf)
    for e in range(model.experts):
        t, k = np.nonzero(idx_r == e)
        order = np.argsort(slot_r[t, k])
        t, k = t[order], k[order]
        gate, up = unpack_w13(w13[e])
        ref = O.expert_ffn(x[t], to_host(gate), to_host(up), to_host(w2[e]))
        assert_close_bf16(ybuf[t, k], ref, f"expert {e} (t_e = {len(t)})")
        y_ref[t, k] = ref
    np.testing.assert_array_equal(to_host(out), O.combine(ybuf, w_r, x))
    assert_close_bf16(to_host(out), O.combine(y_ref, w_r, x), "layer output")
    g.close()


# (name, H, H', totals per local expert, experts checked)
GEMM_SHAPES = [
    ("dbrx", 6144, 10752, [1536, 1101, 0, 643], (0, 1, 3)),
    ("mixtral-8x7b", 4096, 14336, [1536, 1163], (0, 1)),
    ("deepseek-v3", 7168, 2048, None, (0, 17, 40, 41, 63)),
]


@pytest.mark.parametrize("name,H,Hp,totals,check", GEMM_SHAPES, ids=[s[0] for s in GEMM_SHAPES])
def test_grouped_ffn_baseline_shapes(lib, name, H, Hp, totals, check):
    from paper_2504_02263_b200 import ops

    if totals is None:  # E_l = 64 (256 experts over 4 expert GPUs), ragged, some empty / odd-tile
        rng = np.random.default_rng(5)
        totals = rng.integers(0, 400, size=64).tolist()
        totals[17], totals[40], totals[41] = 0, 129, 1
    E_l = len(totals)
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev)
    gen.manual_seed(11)
    gate = (torch.randn((E_l, Hp, H), generator=gen, device=dev) / H ** 0.5).to(torch.bfloat16)
    up = (torch.randn((E_l, Hp, H), generator=gen, device=dev) / H ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn((E_l, H, Hp), generator=gen, device=dev) / Hp ** 0.5).to(torch.bfloat16)
    w13 = ops.pack_w13(gate, up)
    starts = ops.segment_starts(totals)
    rows = max(int(starts[-1]) + (totals[-1] + 127) // 128 * 128, 128)
    x = torch.randn((rows, H), generator=gen, device=dev).to(torch.bfloat16)
    y = ops.grouped_ffn(x, torch.tensor(totals, dtype=torch.int32), w13, w2)
    torch.cuda.synchronize()
    yh, xh = to_host(y), to_host(x)
    for e in check:
        s, t = int(starts[e]), totals[e]
        if t == 0:
            continue
        ref = O.expert_ffn(xh[s:s + t], to_host(gate[e]), to_host(up[e]), to_host(w2[e]))
        assert_close_bf16(yh[s:s + t], ref, f"{name} expert {e} (t_e = {t})")
