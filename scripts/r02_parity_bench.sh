#!/bin/bash
# r02: shape-parity tests, N=1 bench (parity field, full-layer CPU baseline), reference arm
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_shapes.py -q -x > gpurun_out/r02_pytest_shapes.log 2>&1; tail -3 gpurun_out/r02_pytest_shapes.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_n1.json 2> gpurun_out/r02_bench_n1.err; tail -c 600 gpurun_out/r02_bench_n1.err
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref_n1.json 2> gpurun_out/r02_bench_ref_n1.err; tail -c 600 gpurun_out/r02_bench_ref_n1.err
