#!/bin/bash
# CTA-pair epilogue: rows stored from registers + a 7th operand stage vs smem staging (6 stages)
mkdir -p gpurun_out
timeout 300 python scripts/ab_lib_ffn.py scripts/ab_libs/libmsinfer_epistaged.so scripts/ab_libs/libmsinfer_epidirect.so 5 > gpurun_out/ab_epidirect.json 2>&1
timeout 300 python scripts/ab_lib_ffn.py scripts/ab_libs/libmsinfer_epidirect.so scripts/ab_libs/libmsinfer_epistaged.so 5 >> gpurun_out/ab_epidirect.json 2>&1
cat gpurun_out/ab_epidirect.json
