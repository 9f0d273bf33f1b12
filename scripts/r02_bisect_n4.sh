#!/bin/bash
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for envs in "MSI_REGION_RUNS=1" "MSI_FUSED_DISPATCH=0" "MSI_ROUTER_TC=0 MSI_REGION_RUNS=1"; do
  i=$((i+1))
  env $envs DBG_T=2048 timeout -s KILL 120 $R --master-port $((29990 + i)) scripts/dbg_stage_n4.py > /tmp/b.log 2>&1
  echo "[$envs] rc=$? $(grep -c 'combine: status 0' /tmp/b.log) combines ok; last: $(grep '^rank' /tmp/b.log | tail -2 | tr '\n' ' ')"
done
exit 0
