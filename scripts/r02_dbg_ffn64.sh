#!/bin/bash
for cfg in "64 4 64 2048" "64 4 128 2048" "64 1 512 2048" "128 2 128 2048"; do
  set -- $cfg
  AB_SHAPE=deepseek-v3 AB_EL=$1 AB_NSRC=$2 AB_PER=$3 AB_CAP=$4 AB_ITERS=3 timeout -s KILL 60 python scripts/ab_ffn_regions_1gpu.py 2>&1 | tail -1 | cut -c1-250
  echo "cfg $cfg rc=$?"
done
