"""Runtime variants of the tcgen05 GEMM kept as switches must
stay bit-identical to the default CTA-pair kernel: the quad-cluster variant
(MSI_GEMM_QUAD=1, A multicast across two pairs) issues the same MMAs per
tile, so the expert FFN and the dense projections give the same bits on
ragged segments (empty experts, 1-row and odd 128-row tails)."""

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _ffn(ops, cnt, H, Hp, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    E_l = len(cnt)
    rows = sum((c + 127) // 128 * 128 for c in cnt)
    x = torch.randn(rows, H, generator=g, device="cuda").to(torch.bfloat16)
    w13 = ops.pack_w13((torch.randn(E_l, Hp, H, generator=g, device="cuda") / H ** 0.5).to(torch.bfloat16),
                       (torch.randn(E_l, Hp, H, generator=g, device="cuda") / H ** 0.5).to(torch.bfloat16))
    w2 = (torch.randn(E_l, H, Hp, generator=g, device="cuda") / Hp ** 0.5).to(torch.bfloat16)
    tot = torch.tensor(cnt, dtype=torch.int32, device="cuda")
    return lambda: ops.grouped_ffn(x, tot, w13, w2)


@pytest.mark.parametrize("cnt,H,Hp", [([0, 1, 127, 129, 300, 0, 64, 700], 1024, 512),
                                      ([768, 741, 805, 0], 2048, 1024),
                                      ([5, 260, 1000], 6144, 2048)])
def test_quad_cluster_ffn_bit_identical(lib, monkeypatch, cnt, H, Hp):
    from paper_2504_02263_b200 import ops

    run = _ffn(ops, cnt, H, Hp, seed=len(cnt) + H)
    monkeypatch.setenv("MSI_GEMM_QUAD", "0")
    ref = run()
    monkeypatch.setenv("MSI_GEMM_QUAD", "1")
    got = run()
    again = run()
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    assert torch.equal(again, ref)


@pytest.mark.parametrize("T,N,K", [(1, 512, 256), (300, 1536, 1024), (3072, 7680, 6144)])
def test_quad_cluster_dense_bit_identical(lib, monkeypatch, T, N, K):
    from paper_2504_02263_b200 import ops

    g = torch.Generator(device="cuda")
    g.manual_seed(T + N)
    a = torch.randn(T, K, generator=g, device="cuda").to(torch.bfloat16)
    b = (torch.randn(N, K, generator=g, device="cuda") / K ** 0.5).to(torch.bfloat16)
    r = torch.randn(T, N, generator=g, device="cuda").to(torch.bfloat16)
    monkeypatch.setenv("MSI_GEMM_QUAD", "0")
    ref = ops.dense_gemm(a, b, resid=r)
    monkeypatch.setenv("MSI_GEMM_QUAD", "1")
    got = ops.dense_gemm(a, b, resid=r)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
