"""Multi-GPU ping-pong pipeline with the real attention stage: PingPongRunner
on n_a attention GPUs + n_e expert GPUs (one process per GPU), m micro-batches
x L layers chained (x_{l+1} = h_l + MoE(h_l), h_l = attention stage output),
two decode steps.  Each attention rank records its attention outputs and layer
outputs per (layer, micro-batch); the oracle recomputes every layer from the
GPU's own inputs: attention stage within tolerance, then the MoE layer on the
GPU's attention output -- routing bit-exact, output within tolerance
(SURVEY.md §8(e), (f) rank 3).
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


def _host(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def _worker(rank, world, port, n_a, n_e, shape, T, m, L, outdir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2504_02263_b200 import attention as A
    from paper_2504_02263_b200 import ops, runtime
    from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec

    gpu = rank % torch.cuda.device_count()  # fewer GPUs than ranks: share round-robin
    torch.cuda.set_device(gpu)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    model = as_model_spec(shape)
    plan = DeploymentPlan(n_a=n_a, n_e=n_e, m=m, b_a=T)
    g = runtime.M2NGroup(model, plan, rank=rank, device=f"cuda:{gpu}", timeout_s=60)
    wts = O.synth_weights(model.hidden, model.intermediate, model.experts, seed=0)

    def dev(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16).copy()).view(torch.bfloat16).cuda()

    w13 = w2 = wg = None
    if g.is_expert:
        ex = runtime.local_experts(g)
        w13 = ops.pack_w13(dev(wts.w_gate[ex]), dev(wts.w_up[ex]))
        w2 = dev(wts.w_down[ex])
    stages, xs = None, None
    if g.is_attention:
        wg = dev(wts.wg)
        w = A.AttentionWeights(model, f"cuda:{gpu}", seed=5)
        stages = [A.AttentionStage(model, T, L, f"cuda:{gpu}", weights=w, avg_seq_len=80,
                                   seed=100 * g.attn_index + j, headroom=64) for j in range(m)]
        xs = [dev(O.synth_tokens(T, model.hidden, seed=7 * g.attn_index + j)) for j in range(m)]
    layer = runtime.MoEDecodeLayer(g, wg=wg, w13=w13, w2=w2)
    runner = runtime.PingPongRunner(layer, layers=L, attn=stages, chain=True)
    res = {}
    for step in range(2):
        if g.is_attention:
            res[f"x_{step}"] = np.stack([_host(x) for x in xs])
            res[f"ctx_{step}"] = np.stack([st.cache.ctx_host.copy() for st in stages])
            for j, st in enumerate(stages):  # pools differ in size per micro-batch
                res[f"k_{step}_{j}"] = np.stack([_host(st.cache.k[l]) for l in range(L)])
                res[f"v_{step}_{j}"] = np.stack([_host(st.cache.v[l]) for l in range(L)])
            # record each layer's attention output: wrap forward
            rec = {}
            for j, st in enumerate(stages):
                orig = st.forward

                def fwd(x, l, out=None, _st=st, _j=j, _orig=orig):
                    xin = x.clone()
                    y = _orig(x, l, out)
                    rec[(l, _j)] = (y.clone(), xin)
                    return y
                st.forward = fwd
        runner.run(xs)
        torch.cuda.synchronize()
        if g.is_attention:
            torch.cuda.synchronize()
            for j, st in enumerate(stages):
                st.forward = st.__class__.forward.__get__(st)
                st.cache.advance()
            res[f"out_{step}"] = np.stack([_host(x) for x in xs])
            res[f"h_{step}"] = np.stack([np.stack([_host(rec[(l, j)][0]) for j in range(m)]) for l in range(L)])
            res[f"in_{step}"] = np.stack([np.stack([_host(rec[(l, j)][1]) for j in range(m)]) for l in range(L)])
        dist.barrier()
    if g.is_attention:
        res["wqkv"] = _host(stages[0].w.wqkv)
        res["wo"] = _host(stages[0].w.wo)
        for j, st in enumerate(stages):
            res[f"bt_{j}"] = st.cache.block_table_host
        res["theta"] = np.array([stages[0].theta])
        res["heads"] = np.array([stages[0].n_heads, stages[0].n_kv])
    res["status"] = np.array([g.status()])
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **res)
    dist.barrier()
    g.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_a,n_e,T,m,L", [(1, 1, 40, 2, 2), (2, 2, 24, 3, 2)])
def test_pingpong_attention_multi_gpu(lib, tmp_path, n_a, n_e, T, m, L):
    import torch.multiprocessing as mp

    from oracle import oracle as O
    from paper_2504_02263_b200.config import as_model_spec

    world = n_a + n_e
    if torch.cuda.device_count() < world and os.environ.get("MSI_TEST_NO_OVERSUBSCRIBE") == "1":
        pytest.skip(f"needs {world} GPUs")
    model = as_model_spec("tiny")
    mp.spawn(_worker, args=(world, _free_port(), n_a, n_e, "tiny", T, m, L, str(tmp_path)), nprocs=world,
             join=True)
    got = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    for r in range(world):
        assert got[r]["status"][0] == 0
    wts = O.synth_weights(model.hidden, model.intermediate, model.experts, seed=0)
    from _util import assert_close_bf16
    a0 = got[0]
    nh, nkv = (int(v) for v in a0["heads"])
    for step in range(2):
        # every (layer, micro-batch): the oracle attention stage on the GPU's
        # layer input vs the GPU's attention output, then the oracle MoE layer
        # over all senders' GPU attention outputs vs the GPU's layer output
        # (next layer's input, or the final x): routing bit-exact inputs
        for l in range(L):
            for j in range(m):
                hs = []
                for s in range(n_a):
                    a = got[s]
                    kc, vc = a[f"k_{step}_{j}"][l].copy(), a[f"v_{step}_{j}"][l].copy()
                    ref_h = O.attention_stage(a[f"in_{step}"][l][j], a["wqkv"], a["wo"], a[f"ctx_{step}"][j].copy(),
                                              nh, nkv, float(a["theta"][0]), a[f"bt_{j}"], kc, vc)
                    assert_close_bf16(a[f"h_{step}"][l][j], ref_h, f"attention step {step} l {l} rank {s} mb {j}")
                    hs.append(a[f"h_{step}"][l][j])
                ref = O.moe_layer(hs, wts, model.topk, n_e=n_e, resid=True)
                for s in range(n_a):
                    a = got[s]
                    out = a[f"in_{step}"][l + 1][j] if l + 1 < L else a[f"out_{step}"][j]
                    assert_close_bf16(out, ref.out[s], f"layer output step {step} l {l} rank {s} mb {j}")
