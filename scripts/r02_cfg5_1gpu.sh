#!/bin/bash
set -u
mkdir -p gpurun_out
for tc in 1 0; do
  MSI_ROUTER_TC=$tc MSI_BENCH_STACKDUMP=60 timeout -s KILL 150 python bench.py --steps 2 --warmup 2 --no-cpu --no-m2n --no-e2e --shape deepseek-v3 --b-a 2048 --micro-batches 1 > gpurun_out/r02_cfg5_1gpu_tc$tc.log 2>&1
  echo "tc=$tc rc=$?"; grep '^{' gpurun_out/r02_cfg5_1gpu_tc$tc.log | cut -c1-200
  grep -m3 "File \"/tmp" gpurun_out/r02_cfg5_1gpu_tc$tc.log
done
# router-only with dispatch through a co-located 1-rank context at T = 2048, E = 256
cat > /tmp/rd.py <<'PY'
import os, sys, torch
sys.path.insert(0, '.')
from paper_2504_02263_b200 import runtime
from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec
m = as_model_spec("deepseek-v3")
for T in (1024, 2048):
    g = runtime.M2NGroup(m, DeploymentPlan(n_a=1, n_e=1, m=1, b_a=T, colocated=True), rank=0, timeout_s=10)
    wg = runtime.synth_device_weights(m, [], seed=0, device=g.device)[0]
    layer = runtime.MoEDecodeLayer(g, wg=wg)
    x = torch.randn(T, m.hidden, device=g.device).to(torch.bfloat16)
    r = layer.route_dispatch(x, 0)
    torch.cuda.synchronize()
    print(T, "route_dispatch ok, status", g.status(), flush=True)
    g.close()
PY
MSI_ROUTER_TC=1 timeout -s KILL 120 python /tmp/rd.py 2>&1 | tail -5; echo "rd rc=$?"
