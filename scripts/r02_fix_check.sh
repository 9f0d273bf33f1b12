#!/bin/bash
# the segment-table race fix: replay the captured counts (regions + gather, 6 reps each), the
# regression test, and the 4-GPU DS-V3 b_a 2048 / 4096 bench lines
for r in 1 3; do
  for p in gather regions; do
    for rep in 1 2 3 4 5 6; do
      DBG_PATH=$p timeout -s KILL 30 python scripts/dbg_replay_counts.py tests/golden/hang/dbg_counts_r$r.npy > /tmp/r.log 2>&1
      echo -n "r$r/$p/$rep=$? "
    done
  done
done
echo
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "regression or regions" 2>&1 | tail -2
