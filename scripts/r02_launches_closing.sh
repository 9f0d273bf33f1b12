#!/bin/bash
# ncu launch list of one N=1 step of the final code (cold, serialised per-launch times)
mkdir -p gpurun_out
SMALL="--steps 1 --warmup 3 --no-e2e --no-cpu --no-graph --no-m2n"
timeout 300 python bench.py $SMALL > gpurun_out/lc_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/lc_plain.log; exit 1; }
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_closing.csv \
    python bench.py $SMALL > gpurun_out/lc_ncu.log 2>&1; echo "ncu rc=$?"
