#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I include scripts/probe_mma_rate.cu -o gpurun_out/probe_mma_rate && timeout 120 gpurun_out/probe_mma_rate | tee gpurun_out/probe_mma_rate.jsonl
