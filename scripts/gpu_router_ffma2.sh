#!/bin/bash
# Router with packed FFMA2 logits: bit-exact router tests (fused, split and
# every tile override), router microbench, and the N = 1 bench.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k router > gpurun_out/f2_pytest.log 2>&1; tail -n 1 gpurun_out/f2_pytest.log
MSI_ROUTER_SPLIT=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k router > gpurun_out/f2_pytest_fused.log 2>&1; tail -n 1 gpurun_out/f2_pytest_fused.log
for tile in 8x8x32 2x8x16 4x4x16 1x16x8; do
  MSI_ROUTER_TILE=$tile timeout 600 python -m pytest tests/test_gpu_parity.py -q -k router_bit_exact > gpurun_out/f2_pytest_$tile.log 2>&1; echo "tile $tile: $(tail -n 1 gpurun_out/f2_pytest_$tile.log)"
done
for r in 1 2; do timeout 300 python scripts/bench_router.py 2>&1 | grep '^{'; done | tee gpurun_out/f2_router_bench.txt
timeout 600 python bench.py > gpurun_out/f2_bench_n1.log 2>&1; grep '^{' gpurun_out/f2_bench_n1.log | tail -n 1 > gpurun_out/f2_bench_n1.json
python -c "
import json; d=json.load(open('gpurun_out/f2_bench_n1.json')); print(round(d['value']), d['e2e']['value'], d['roofline']['frac'])"
