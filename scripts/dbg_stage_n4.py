#!/usr/bin/env python
"""Stage-by-stage M2N + FFN with status checks (torchrun, co-located ranks)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
from paper_2504_02263_b200 import runtime
from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec

rank, world, local = runtime.init_distributed_from_env("nccl")
m = as_model_spec(os.environ.get("DBG_SHAPE", "deepseek-v3"))
T = int(os.environ.get("DBG_T", "2048"))
g = runtime.M2NGroup(m, DeploymentPlan(n_a=world, n_e=world, m=1, b_a=T, colocated=True), rank=rank, timeout_s=5)
wg, w13, w2 = runtime.synth_device_weights(m, runtime.local_experts(g), seed=0, device=g.device)
layer = runtime.MoEDecodeLayer(g, wg=wg, w13=w13, w2=w2)
x = torch.randn(T, m.hidden, device=g.device).to(torch.bfloat16)
def st(tag):
    torch.cuda.synchronize()
    s = g.status()
    print(f"rank {rank} {tag}: status {s}", flush=True)
    dist.barrier()
for it in range(2):
    r = layer.route_dispatch(x, 0); st(f"it{it} route_dispatch")
    layer.expert_wait(0); st(f"it{it} expert_wait")
    if it == 0:
        import numpy as np
        tab = (g.cntab_view(0).cpu().numpy() & 0xffffffff).astype(np.int64)  # [n_a][E]
        E_l = m.experts // world
        np.save(f"gpurun_out/dbg_counts_r{rank}.npy", tab[:, rank * E_l:(rank + 1) * E_l])
    layer.expert_ffn(0); st(f"it{it} expert_ffn")
    layer.combine(r); st(f"it{it} combine")
g.close()
dist.destroy_process_group()
