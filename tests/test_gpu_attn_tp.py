"""Attention-node tensor parallelism (DeploymentPlan.tp_a > 1; PAPER.md:192,
441-443; csrc/attn_tp.cu): tp_a processes, one per GPU (sharing GPUs
round-robin on a smaller box), each with its own token shard and 1/tp_a of
the heads.  The node's output shards are compared with the CPU oracle's
attention stage over all node tokens with the full weights and the full KV
cache (assembled from the GPUs' head slices).

Tolerance (floating point, stated here): rel-L2 <= 5e-3 and max-abs <=
2^-7 max|ref| (tests/_util.py) -- the partial O-projection rows are rounded to
bf16 before the fp32 reduce, one more rounding than the oracle.  Index work is
exact: the appended cache rows land at (page of pos, pos % 64) of this GPU's
KV heads.  A second use of the same micro-batch slot (epoch 2) gives the
bit-identical output.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _u16(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def _worker(rank, world, port, spec, T, ctx_lens, outdir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2504_02263_b200 import attention as A
    from paper_2504_02263_b200 import runtime
    from paper_2504_02263_b200.config import DeploymentPlan, MoeModelSpec

    gpu = rank % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    model = MoeModelSpec(**spec)
    plan = DeploymentPlan(n_a=world, n_e=world, m=2, b_a=T, colocated=True, tp_a=world)
    g = runtime.M2NGroup(model, plan, rank=rank, device=f"cuda:{gpu}", timeout_s=60)
    w = A.AttentionWeights(model, g.device, seed=0)
    res = {}
    for slot in range(2):
        st = A.AttentionTPStage(model, T, 1, g, slot, w, np.asarray(ctx_lens, np.int32), seed=7 + slot)
        res[f"k0_{slot}"] = _u16(st.cache.k[0])
        res[f"v0_{slot}"] = _u16(st.cache.v[0])
        x = O.synth_tokens(T, model.hidden, seed=100 * slot + rank)
        xd = torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).cuda()
        y = st.forward(xd, 0).clone()
        y2 = st.forward(xd, 0, out=torch.empty_like(xd))  # second use of the slot (epoch 2), same cache rows
        torch.cuda.synchronize()
        res[f"y_{slot}"] = _u16(y)
        res[f"y2_{slot}"] = _u16(y2)
        res[f"k1_{slot}"] = _u16(st.cache.k[0])
        res[f"v1_{slot}"] = _u16(st.cache.v[0])
        res[f"bt_{slot}"] = st.cache.block_table_host
        if rank == 0:
            res[f"wqkv"] = _u16(w.wqkv)
            res[f"wo"] = _u16(w.wo)
        dist.barrier()
    res["status"] = np.array([g.status()])
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **res)
    dist.barrier()
    g.close()
    dist.destroy_process_group()


CASES = [
    # tp_a, model spec (n_heads = hidden/128, gqa_group), T per GPU
    (2, dict(name="tp2", layers=1, hidden=1024, intermediate=512, experts=8, topk=2, gqa_group=2), 37),
    (4, dict(name="tp4", layers=1, hidden=1024, intermediate=512, experts=8, topk=2, gqa_group=2), 20),
    (2, dict(name="tp2-8x22b", layers=1, hidden=6144, intermediate=16384, experts=8, topk=2, gqa_group=8), 9),
]


@pytest.mark.parametrize("tp,spec,T", CASES)
def test_attention_tp_vs_oracle(lib, tmp_path, tp, spec, T):
    import torch.multiprocessing as mp

    from oracle import oracle as O
    from paper_2504_02263_b200.attention import ROPE_THETA, head_layout
    from paper_2504_02263_b200.config import MoeModelSpec

    from _util import assert_close_bf16

    rng = np.random.default_rng(tp * 100 + T)
    ctx = rng.integers(0, 300, size=tp * T).astype(np.int32)
    ctx[:3] = [0, 63, 64]
    port = _free_port()
    mp.spawn(_worker, args=(tp, port, spec, T, ctx.tolist(), str(tmp_path)), nprocs=tp, join=True)
    got = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(tp)]
    for r in range(tp):
        assert got[r]["status"][0] == 0, f"rank {r} device status {got[r]['status']}"
    model = MoeModelSpec(**spec)
    n_heads, n_kv = head_layout(model)
    kl = n_kv // tp
    for slot in range(2):
        bt = got[0][f"bt_{slot}"]
        for r in range(tp):
            np.testing.assert_array_equal(got[r][f"bt_{slot}"], bt)  # one block table per node
        k = np.concatenate([got[r][f"k0_{slot}"] for r in range(tp)], axis=1)  # [pages, n_kv, 64, 128]
        v = np.concatenate([got[r][f"v0_{slot}"] for r in range(tp)], axis=1)
        x = np.concatenate([O.synth_tokens(T, model.hidden, seed=100 * slot + r) for r in range(tp)])
        ref = O.attention_stage(x, got[0]["wqkv"], got[0]["wo"], ctx.copy(), n_heads, n_kv, ROPE_THETA, bt, k, v)
        for r in range(tp):
            assert_close_bf16(got[r][f"y_{slot}"], ref[r * T:(r + 1) * T], f"tp={tp} slot={slot} shard {r}")
            np.testing.assert_array_equal(got[r][f"y2_{slot}"], got[r][f"y_{slot}"])
            # the appended rows: this GPU's KV heads, exact positions, values within tolerance
            k1, k0 = got[r][f"k1_{slot}"], got[r][f"k0_{slot}"]
            changed = {(int(pg), int(rr)) for pg, _, rr in np.argwhere((k1 != k0).any(axis=-1))}
            want = {(int(bt[t, ctx[t] // 64]), int(ctx[t] % 64)) for t in range(tp * T)}
            assert changed <= want
            rows_g = np.stack([k1[bt[t, ctx[t] // 64], :, ctx[t] % 64] for t in range(tp * T)])
            rows_r = np.stack([k[bt[t, ctx[t] // 64], r * kl:(r + 1) * kl, ctx[t] % 64] for t in range(tp * T)])
            assert_close_bf16(rows_g, rows_r, f"appended k rows, shard {r}")


def _runner_worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2504_02263_b200 import attention as A
    from paper_2504_02263_b200 import ops, runtime
    from paper_2504_02263_b200.config import DeploymentPlan, MoeModelSpec

    gpu = rank % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    model = MoeModelSpec("tpr", 2, 1024, 512, 8, 2, gqa_group=2)
    T, m, L = 24, 2, 2
    plan = DeploymentPlan(n_a=2, n_e=1, m=m, b_a=T, tp_a=2)  # one attention node of 2 GPUs + 1 expert GPU
    g = runtime.M2NGroup(model, plan, rank=rank, device=f"cuda:{gpu}", timeout_s=60)
    wts = O.synth_weights(model.hidden, model.intermediate, model.experts, seed=0)

    def dev(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16).copy()).view(torch.bfloat16).cuda()

    layer_kw = {}
    stages = None
    xs = None
    if g.is_expert:
        ex = runtime.local_experts(g)
        layer_kw = dict(w13=ops.pack_w13(dev(wts.w_gate[ex]), dev(wts.w_up[ex])), w2=dev(wts.w_down[ex]))
    if g.is_attention:
        w = A.AttentionWeights(model, g.device, seed=0)
        ctx = np.arange(2 * T, dtype=np.int32) * 7 % 200
        stages = [A.AttentionTPStage(model, T, L, g, j, w, ctx, seed=3 + j) for j in range(m)]
        layer_kw = dict(wg=dev(wts.wg))
        xs = [dev(O.synth_tokens(T, model.hidden, seed=50 * j + g.attn_index)) for j in range(m)]
    layer = runtime.MoEDecodeLayer(g, **layer_kw)
    runner = runtime.PingPongRunner(layer, layers=L, chain=False, attn=stages)
    dist.barrier()
    runner.run(xs)
    torch.cuda.synchronize()
    res = {}
    if g.is_attention:
        res["eager"] = np.stack([_u16(runner._out(xs, j)) for j in range(m)])
    dist.barrier()
    runner.capture(xs)  # device-tracked epochs for the TP kernels too
    for _ in range(2):
        runner.replay()
    torch.cuda.synchronize()
    if g.is_attention:
        res["graph"] = np.stack([_u16(runner._out(xs, j)) for j in range(m)])
        r = layer._routes[0]
        h = stages[0].y[:T]
        idx_r, w_r = O.router(_u16(h), wts.wg, model.topk)
        res["routing_ok"] = np.array([np.array_equal(r.idx[:T].cpu().numpy(), idx_r)])
    res["status"] = np.array([g.status()])
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **res)
    dist.barrier()
    g.close()
    dist.destroy_process_group()


def test_attention_tp_in_pingpong_runner_with_graph(lib, tmp_path):
    """PingPongRunner on one attention node of 2 GPUs (tp_a = 2) + 1 expert
    GPU, 2 micro-batches x 2 layers, eager then CUDA-graph replays (the TP
    kernels' device-tracked epochs): every status 0, the graph replays give
    the eager step's outputs bit for bit, routing of the TP stage's output
    bit-exact vs the oracle."""
    import torch.multiprocessing as mp

    mp.spawn(_runner_worker, args=(3, _free_port(), str(tmp_path)), nprocs=3, join=True)
    got = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(3)]
    for r in range(3):
        assert got[r]["status"][0] == 0, r
    for r in range(2):  # attention ranks
        np.testing.assert_array_equal(got[r]["graph"], got[r]["eager"])
        assert got[r]["routing_ok"][0]
