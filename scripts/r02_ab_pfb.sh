#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/ab_pfb.py > gpurun_out/ab_pfb.jsonl 2>&1; echo "rc=$?"; cat gpurun_out/ab_pfb.jsonl
