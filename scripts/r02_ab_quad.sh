#!/bin/bash
mkdir -p gpurun_out
timeout 240 python scripts/ab_quad.py > gpurun_out/ab_quad.jsonl 2>&1; echo "rc=$?"; cat gpurun_out/ab_quad.jsonl | tail -12
