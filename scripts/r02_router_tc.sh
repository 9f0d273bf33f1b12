#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "router" > gpurun_out/r02_pytest_router_tc.log 2>&1; tail -15 gpurun_out/r02_pytest_router_tc.log | cut -c1-300
timeout 600 python scripts/ab_router_tc.py > gpurun_out/r02_ab_router_tc.jsonl 2> gpurun_out/r02_ab_router_tc.err; cat gpurun_out/r02_ab_router_tc.jsonl; tail -3 gpurun_out/r02_ab_router_tc.err
