#!/usr/bin/env python
"""Same-box A/B of the expert FFN with several senders (torchrun, co-located
N ranks, Mixtral-8x22B, T tokens per rank): msi_expert_ffn reading A as runs
of the (expert, sender) receive regions vs msi_grouped_ffn on the same rows
packed compactly per expert (one run per tile).  Medians per rank."""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2504_02263_b200 import ops, runtime  # noqa: E402
from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    rank, world, local = runtime.init_distributed_from_env("nccl")
    model = as_model_spec(os.environ.get("AB_SHAPE", "mixtral-8x22b"))
    T = int(os.environ.get("AB_T", "3072"))
    plan = DeploymentPlan(n_a=world, n_e=world, m=1, b_a=T, colocated=True)
    g = runtime.M2NGroup(model, plan, rank=rank)
    wg, w13, w2 = runtime.synth_device_weights(model, runtime.local_experts(g), seed=0, device=g.device)
    layer = runtime.MoEDecodeLayer(g, wg=wg, w13=w13, w2=w2)
    gen = torch.Generator(device=g.device)
    gen.manual_seed(1 + rank)
    x = torch.randn(T, model.hidden, generator=gen, device=g.device).to(torch.bfloat16)
    E_l = model.experts // world

    def round_trip(timed):
        dist.barrier()
        r = layer.route_dispatch(x, 0)
        layer.expert_wait(0)
        s, e = ev(), ev()
        s.record()
        layer.expert_ffn(0)
        e.record()
        layer.combine(r)
        torch.cuda.synchronize()
        return s.elapsed_time(e)

    for _ in range(3):
        round_trip(False)
    tab = g.cntab_view(0).cpu()
    cnt = [[int(tab[s, rank * E_l + e]) & 0xffffffff for e in range(E_l)] for s in range(world)]
    tot = [sum(cnt[s][e] for s in range(world)) for e in range(E_l)]
    starts = ops.segment_starts(tot)
    rows = starts[-1] + (tot[-1] + 127) // 128 * 128
    recv = g.recv_view(0)
    xc = torch.zeros(rows, model.hidden, dtype=torch.bfloat16, device=g.device)
    for e in range(E_l):
        o = starts[e]
        for s in range(world):
            base = (e * world + s) * T
            xc[o:o + cnt[s][e]] = recv[base: base + cnt[s][e]]
            o += cnt[s][e]
    tt = torch.tensor(tot, dtype=torch.int32, device=g.device)
    hbuf = torch.empty(rows, model.intermediate, dtype=torch.bfloat16, device=g.device)
    y = torch.empty(rows, model.hidden, dtype=torch.bfloat16, device=g.device)
    flops = 6.0 * sum(tot) * model.hidden * model.intermediate
    res = {"regions_ms": [], "compact_ms": []}
    for _ in range(int(os.environ.get("AB_ITERS", "10"))):
        res["regions_ms"].append(round_trip(True))
        c0, c1 = ev(), ev()
        c0.record()
        ops.grouped_ffn(xc, tt, w13, w2, hbuf, y)
        c1.record()
        torch.cuda.synchronize()
        res["compact_ms"].append(c0.elapsed_time(c1))
    assert g.status() == 0
    out = {k: statistics.median(v) for k, v in res.items()}
    out["regions_tflops"] = flops / (out["regions_ms"] * 1e-3) / 1e12
    out["compact_tflops"] = flops / (out["compact_ms"] * 1e-3) / 1e12
    out.update(rank=rank, world=world, shape=model.name, T=T, counts=cnt,
               cg=os.environ.get("MSI_GEMM_CG", "2"))
    allo = [None] * world
    dist.all_gather_object(allo, out)
    if rank == 0:
        for o in allo:
            print(json.dumps(o), flush=True)
    g.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
