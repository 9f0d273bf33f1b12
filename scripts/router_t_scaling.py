import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
from paper_2504_02263_b200 import ops
H,E,K=6144,8,2
for T in (32, 96, 256, 1024, 3072):
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    wg = (torch.randn(E, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
    ws = ops.RouterWorkspace(T, E, "cuda")
    for _ in range(5): ops.gate_topk(x, wg, K, ws=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for _ in range(20): ops.gate_topk(x, wg, K, ws=ws)
    torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); torch.cuda.synchronize()
    print(json.dumps({"T":T,"us_graph":a.elapsed_time(b)/20*1e3}))
