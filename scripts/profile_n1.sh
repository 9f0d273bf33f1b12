#!/bin/bash
# One-GPU measurement pass (run under gpurun from the repo root):
#  1. the default bench line (no profiler)            -> gpurun_out/bench_n1.json
#  2. ncu launch list of the same command (cold, serialised per-launch times)
#                                                      -> gpurun_out/launches_n1.csv
#  3. ncu --set full of one GEMM1/GEMM2 pair and one decode-attention launch
#                                                      -> gpurun_out/full_*.ncu-rep
# Each ncu pass runs only after the plain command exited 0.
set -u
mkdir -p gpurun_out
ARGS="--steps ${STEPS:-10} --warmup ${WARMUP:-3}"
timeout 600 python bench.py $ARGS --timeline-csv gpurun_out/timeline_n1_r{rank}.csv > gpurun_out/bench_n1.log 2>&1 || { echo "bench failed"; tail -20 gpurun_out/bench_n1.log; exit 1; }
grep '^{' gpurun_out/bench_n1.log | tail -1 > gpurun_out/bench_n1.json
NCU=/usr/local/cuda/bin/ncu
SMALL="--steps 1 --warmup 3 --no-e2e --no-cpu --no-graph --no-m2n"
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv \
    python bench.py $SMALL > gpurun_out/ncu_launches.log 2>&1 || echo "launch list failed"
# grouped_gemm launches per layer: QKV (+RoPE/append), O projection, GEMM1, GEMM2
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:grouped_gemm -s 26 -c 2 \
    -o gpurun_out/full_gemm -f python bench.py $SMALL > gpurun_out/ncu_gemm.log 2>&1 || echo "gemm capture failed"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:grouped_gemm -s 24 -c 2 \
    -o gpurun_out/full_proj -f python bench.py $SMALL > gpurun_out/ncu_proj.log 2>&1 || echo "proj capture failed"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:decode_attn -s 12 -c 1 \
    -o gpurun_out/full_attn -f python bench.py $SMALL > gpurun_out/ncu_attn.log 2>&1 || echo "attn capture failed"
python scripts/summarize_launches.py gpurun_out/launches_n1.csv 4 "N=1 launch list" > gpurun_out/launches_n1_summary.txt 2>&1
cat gpurun_out/launches_n1_summary.txt
ls -la gpurun_out/
