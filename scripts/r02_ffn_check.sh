#!/bin/bash
# FFN / projections / N=1 bench check after a GEMM kernel change
set -u
mkdir -p gpurun_out
for n in 1 2; do per=$((1536 / n)); AB_NSRC=$n AB_PER=$per timeout 300 python scripts/ab_ffn_regions_1gpu.py 2>/dev/null | cut -c1-260; done
timeout 300 python scripts/ab_dense_gemm.py 2>/dev/null | head -1 | cut -c1-400
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --timeline-csv gpurun_out/tl_chk.csv > gpurun_out/r02_bench_n1_chk.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/r02_bench_n1_chk.json')); print(int(d['value']), round(d['roofline']['achieved']), d['stage_times']['T_a_ms'], d['stage_times']['T_e_ms'], d['clocks']['sm_mhz'])"
