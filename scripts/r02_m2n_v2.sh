#!/bin/bash
# r02: receive regions + fused router/dispatch: GPU suite, then N=1 bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_build.log 2>&1 || { tail -20 gpurun_out/r02_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_v2.log 2>&1; tail -15 gpurun_out/r02_pytest_v2.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r02_bench_n1_v2.json 2> gpurun_out/r02_bench_n1_v2.err; tail -c 400 gpurun_out/r02_bench_n1_v2.err
