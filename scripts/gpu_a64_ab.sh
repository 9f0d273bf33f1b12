#!/bin/bash
# Half-pair 64-row A box A/B (1 GPU): GEMM parity tests, interleaved GEMM A/B
# (MSI_GEMM_A64=0 : 1) over ragged t_e, and the N=1 bench alternating.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_attention.py -q -x > gpurun_out/pytest_a64.log 2>&1; tail -2 gpurun_out/pytest_a64.log
timeout 900 python bench_gemm.py --ab 6 --ab-env MSI_GEMM_A64=0:1 --te 256,512,768,1024,1536 --iters 5 > gpurun_out/gemm_a64_ab.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/gemm_a64_ab.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['te'], d['odd_tiles'], round(d['cg1_tflops']), '->', round(d['cg2_tflops']), round(d['cg2_over_cg1'],3))
"
for A in 0 1 0 1; do
  MSI_GEMM_A64=$A timeout 300 python bench.py --no-cpu --no-e2e --no-m2n --steps 20 > gpurun_out/bench_a64_$A.log 2>&1
  grep '^{' gpurun_out/bench_a64_$A.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('A64', $A, round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
done
