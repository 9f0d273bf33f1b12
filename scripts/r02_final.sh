#!/bin/bash
# final validation on the final code (one GPU): GPU suite (multi-rank plans share the GPU),
# smoke, N=1 bench line, reference arm
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_final.log 2>&1; tail -3 gpurun_out/r02_pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_n1_last.json 2> gpurun_out/r02_bench_n1_last.err; tail -c 200 gpurun_out/r02_bench_n1_last.err
python -c "
import json; d=json.load(open('gpurun_out/r02_bench_n1_last.json')); print(int(d['value']), int(d['e2e']['value']), round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['cpu_baseline']['value'], d['clocks']['sm_mhz'], d['parity']['routing_bit_exact'], d['gpu_launches'])"
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02_bench_ref_last.json 2>/dev/null; head -c 300 gpurun_out/r02_bench_ref_last.json
