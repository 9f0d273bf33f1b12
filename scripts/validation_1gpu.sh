#!/bin/bash
# Round-end re-validation on a 1-GPU box: GPU suite, smoke, bench N = 1.
set -u
mkdir -p gpurun_out
MSI_TEST_OVERSUBSCRIBE=1 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/v1_pytest_gpu.log 2>&1; tail -3 gpurun_out/v1_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v1_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/v1_smoke.log
timeout 600 python bench.py > gpurun_out/v1_bench_n1.log 2>&1; grep '^{' gpurun_out/v1_bench_n1.log | tail -1 > gpurun_out/v1_bench_n1.json
python -c "
import json; d=json.load(open('gpurun_out/v1_bench_n1.json')); print(round(d['value']), d['e2e']['value'], d['roofline']['frac'], d['m2n']['p50_us'], d['clocks'])"
