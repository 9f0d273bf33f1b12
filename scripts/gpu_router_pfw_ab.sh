#!/bin/bash
# A/B of the L1 prefetch of the next W_g chunk in the router logits loop
# (MSI_ROUTER_PFW); parity tests run with it on.
set -u
mkdir -p gpurun_out
MSI_ROUTER_PFW=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k router > gpurun_out/pfw_pytest.log 2>&1; tail -2 gpurun_out/pfw_pytest.log
MSI_ROUTER_SPLIT=0 MSI_ROUTER_PFW=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k router > gpurun_out/pfw_pytest_fused.log 2>&1; tail -1 gpurun_out/pfw_pytest_fused.log
for r in 1 2; do
for v in 0 1; do
  echo "== MSI_ROUTER_PFW=$v (rep $r)"
  MSI_ROUTER_PFW=$v timeout 300 python scripts/bench_router.py 2>&1 | grep '^{'
done; done | tee gpurun_out/pfw_ab.txt
