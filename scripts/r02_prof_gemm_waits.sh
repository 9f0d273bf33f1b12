#!/bin/bash
mkdir -p gpurun_out
for sh in "8 768" "4 1536" "8 384"; do timeout 300 python scripts/prof_gemm_waits.py scripts/ab_libs/libmsinfer_gemmprof.so $sh; done 2>&1 | tee gpurun_out/prof_gemm_waits.jsonl
