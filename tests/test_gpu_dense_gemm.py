"""The attention stage's projections on the tcgen05 GEMM (PAPER.md:283-284,
Table 3 "QKV Project" / "Attn Output"): msi_dense_gemm (O projection with the
residual in the epilogue) and msi_qkv_rope_append (QKV projection with RoPE
and the paged-KV append in the epilogue).

Tolerance (floating point, stated here): bf16 outputs within rel-L2 <= 5e-3
and max-abs <= 2^-7 * max|ref| of a plain torch fp32 reference of the same
op (fp32 accumulation of the bf16 operands, one bf16 rounding; tests/_util.py).
Index work is exact: the fused QKV epilogue must write exactly the cache rows
(page, KV head, pos % 64) the oracle's rope_append writes, and nothing else.
The fused kernel is also compared with the unfused GPU path (dense GEMM ->
msi_rope_append): same MMAs, same rotation arithmetic -> bit-identical.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

from _util import assert_close_bf16  # noqa: E402


def u16(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def bf16_randn(shape, gen, scale=1.0):
    return (torch.randn(shape, generator=gen, device="cuda") * scale).to(torch.bfloat16)


DENSE_CASES = [
    # T, N, K
    (1, 256, 64),
    (5, 768, 512),
    (127, 512, 512),
    (130, 512, 1024),
    (257, 1280, 1024),
    (1000, 7680, 6144),   # Mixtral-8x22B QKV at b_a = 1000 (ragged tail tile)
    (3072, 6144, 6144),   # Mixtral-8x22B O projection at the N = 1 bench batch
]


@pytest.mark.parametrize("T,N,K", DENSE_CASES)
@pytest.mark.parametrize("resid", [False, True])
def test_dense_gemm_vs_torch_fp32(lib, T, N, K, resid):
    from paper_2504_02263_b200 import ops

    g = torch.Generator(device="cuda")
    g.manual_seed(T * 7 + N + K)
    a = bf16_randn((T, K), g)
    b = bf16_randn((N, K), g, K ** -0.5)
    r = bf16_randn((T, N + 64), g)[:, :N] if resid else None  # padded row stride
    out = torch.full((T, N + 128), float("nan"), dtype=torch.bfloat16, device="cuda")
    ops.dense_gemm(a, b, out[:, :N], resid=r)
    torch.cuda.synchronize()
    ref = a.float() @ b.float().t()
    if resid:
        ref = ref + r.float()
    assert_close_bf16(u16(out[:, :N]), u16(ref.to(torch.bfloat16)), f"dense_gemm {T}x{N}x{K}")
    assert torch.isnan(out[:, N:].float()).all(), "wrote past N"


def test_dense_gemm_back_to_back_counter_reuse(lib):
    """One tile counter serves consecutive launches on a stream (each launch
    leaves it at 0), including an empty one."""
    from paper_2504_02263_b200 import ops

    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    ctr = ops.TileCounter(1)
    a = bf16_randn((300, 512), g)
    b = bf16_randn((768, 512), g, 512 ** -0.5)
    outs = [ops.dense_gemm(a, b, ctr=ctr) for _ in range(3)]
    ops.dense_gemm(a[:0], b, torch.empty((0, 768), dtype=torch.bfloat16, device="cuda"), ctr=ctr)
    outs.append(ops.dense_gemm(a, b, ctr=ctr))
    torch.cuda.synchronize()
    assert int(ctr.buf[0]) == 0
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def make_cache(T, n_kv, pos, seed):
    rng = np.random.default_rng(seed)
    need = [(p + 1 + 63) // 64 for p in pos]
    npages = sum(need)
    perm = rng.permutation(npages).astype(np.int32)
    bt = np.zeros((T, max(need)), np.int32)
    off = 0
    for t in range(T):
        bt[t, : need[t]] = perm[off: off + need[t]]
        off += need[t]
    k = O.bf16_round(rng.standard_normal((npages, n_kv, 64, 128), dtype=np.float32))
    v = O.bf16_round(rng.standard_normal((npages, n_kv, 64, 128), dtype=np.float32))
    return k, v, bt


def dev(a_u16):
    return torch.from_numpy(np.ascontiguousarray(a_u16).view(np.int16).copy()).view(torch.bfloat16).cuda()


QKV_CASES = [
    # T, hidden, n_heads, n_kv
    (9, 512, 4, 1),        # tiny (G = 4): 6 heads = 3 N tiles
    (70, 2048, 16, 2),     # G = 8, half-pair tail (70 rows)
    (200, 6144, 48, 6),    # Mixtral-8x22B heads: 60 heads = 30 N tiles
    (131, 4096, 32, 4),    # Mixtral-8x7B heads
]


@pytest.mark.parametrize("T,H,n_heads,n_kv", QKV_CASES)
def test_qkv_rope_append_vs_oracle(lib, T, H, n_heads, n_kv):
    from paper_2504_02263_b200 import ops

    rng = np.random.default_rng(T + H)
    pos = rng.integers(0, 1500, size=T).astype(np.int32)
    pos[: min(T, 4)] = [0, 63, 64, 127][: min(T, 4)]  # page edges
    k, v, bt = make_cache(T, n_kv, pos, seed=T)
    x = O.bf16_round(rng.standard_normal((T, H), dtype=np.float32))
    width = (n_heads + 2 * n_kv) * 128
    wqkv = O.bf16_round(rng.standard_normal((width, H), dtype=np.float32) / np.sqrt(H))
    # oracle: qkv = bf16(x wqkv^T) in fp32, then rope_append (caches in place)
    qkv = O.bf16_round(O.bf16_to_f32(x) @ O.bf16_to_f32(wqkv).T)
    k_ref, v_ref = k.copy(), v.copy()
    q_ref = O.rope_append(qkv, pos, n_heads, n_kv, 1e6, bt, k_ref, v_ref)
    kd, vd = dev(k), dev(v)
    q_out = torch.empty((T, n_heads, 128), dtype=torch.bfloat16, device="cuda")
    ops.qkv_rope_append(dev(x), dev(wqkv), torch.from_numpy(pos).cuda(), n_heads, n_kv, 1e6,
                        torch.from_numpy(bt).cuda(), kd, vd, q_out)
    torch.cuda.synchronize()
    assert_close_bf16(u16(q_out).reshape(T, -1), q_ref.reshape(T, -1), "fused rope q")
    kg, vg = u16(kd), u16(vd)
    # exactly the appended rows changed (index work is exact)
    rows = {(int(bt[t, pos[t] // 64]), int(pos[t] % 64)) for t in range(T)}
    for cache, orig in ((kg, k), (vg, v)):
        changed = {(int(pg), int(r)) for pg, _, r in np.argwhere((cache != orig).any(axis=-1))}
        assert changed <= rows
    sel_g_k = np.stack([kg[bt[t, pos[t] // 64], :, pos[t] % 64] for t in range(T)])
    sel_r_k = np.stack([k_ref[bt[t, pos[t] // 64], :, pos[t] % 64] for t in range(T)])
    sel_g_v = np.stack([vg[bt[t, pos[t] // 64], :, pos[t] % 64] for t in range(T)])
    sel_r_v = np.stack([v_ref[bt[t, pos[t] // 64], :, pos[t] % 64] for t in range(T)])
    assert_close_bf16(sel_g_k, sel_r_k, "fused rope k rows")
    assert_close_bf16(sel_g_v, sel_r_v, "fused v rows")


def test_qkv_rope_append_equals_unfused_gpu_path(lib):
    """Fused epilogue == dense GEMM to a qkv buffer + msi_rope_append, bit for bit."""
    from paper_2504_02263_b200 import ops

    T, H, n_heads, n_kv = 300, 2048, 16, 2
    rng = np.random.default_rng(5)
    pos = rng.integers(0, 900, size=T).astype(np.int32)
    k, v, bt = make_cache(T, n_kv, pos, seed=1)
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    x = bf16_randn((T, H), g)
    wqkv = bf16_randn(((n_heads + 2 * n_kv) * 128, H), g, H ** -0.5)
    posd, btd = torch.from_numpy(pos).cuda(), torch.from_numpy(bt).cuda()
    k1, v1, k2, v2 = dev(k), dev(v), dev(k), dev(v)
    q1 = torch.empty((T, n_heads, 128), dtype=torch.bfloat16, device="cuda")
    q2 = torch.empty_like(q1)
    ops.qkv_rope_append(x, wqkv, posd, n_heads, n_kv, 1e6, btd, k1, v1, q1)
    qkv = ops.dense_gemm(x, wqkv)
    ops.rope_append(qkv, posd, n_heads, n_kv, 1e6, btd, k2, v2, q2)
    torch.cuda.synchronize()
    assert torch.equal(q1.view(torch.int16), q2.view(torch.int16))
    assert torch.equal(k1.view(torch.int16), k2.view(torch.int16))
    assert torch.equal(v1.view(torch.int16), v2.view(torch.int16))


@pytest.mark.parametrize("T,E,H", [(5, 256, 512), (130, 256, 7168), (1000, 512, 4096)])
def test_dense_logits_fp32_vs_torch(lib, T, E, H):
    """The router's tensor-core candidate logits (fp32 out) vs torch fp32:
    within the fp32 summation bound used by the router (4 H 2^-24 |x| |w|)."""
    from paper_2504_02263_b200 import ops

    g = torch.Generator(device="cuda")
    g.manual_seed(T + E)
    x = bf16_randn((T, H), g)
    wg = bf16_randn((E, H), g, H ** -0.5)
    got = ops.dense_logits(x, wg)
    torch.cuda.synchronize()
    ref = (x.double() @ wg.double().t())
    bound = 4 * H * 2.0 ** -24 * x.double().norm(dim=1, keepdim=True) * wg.double().norm(dim=1)[None, :]
    assert ((got.double() - ref).abs() <= bound).all()
    assert (got.double() - ref).abs().max() < 1e-3
