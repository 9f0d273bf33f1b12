#!/bin/bash
# r02 1-GPU validation of HEAD: GPU suite (multi-rank tests share the GPU), smoke, N=1 bench
set -u
mkdir -p gpurun_out
T=${TAG:-v}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_$T.log 2>&1; tail -15 gpurun_out/r02_pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_$T.log 2>&1; tail -3 gpurun_out/r02_smoke_$T.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r02_bench_n1_$T.json 2> gpurun_out/r02_bench_n1_$T.err; tail -c 600 gpurun_out/r02_bench_n1_$T.err; cat gpurun_out/r02_bench_n1_$T.json | head -c 3000
