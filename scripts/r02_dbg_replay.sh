#!/bin/bash
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
DBG_T=2048 timeout -s KILL 90 $R --master-port 29995 scripts/dbg_stage_n4.py > /tmp/b.log 2>&1
grep -a '^rank' /tmp/b.log | tail -6
sleep 5
for r in 0 1 2 3; do
  for p in gather regions; do
    DBG_PATH=$p timeout -s KILL 40 python scripts/dbg_replay_counts.py gpurun_out/dbg_counts_r$r.npy > /tmp/r.log 2>&1
    echo "rank $r $p rc=$? $(cat /tmp/r.log | tr '\n' ' ' | cut -c1-150)"
  done
done
python -c "
import numpy as np
for r in range(4):
    c = np.load(f'gpurun_out/dbg_counts_r{r}.npy'); t = c.sum(0)
    print(r, c.shape, 'per-region min/max', c.min(), c.max(), 'tot', t.min(), t.max())"
exit 0
