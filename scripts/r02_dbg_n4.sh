#!/bin/bash
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
DBG_T=2048 timeout -s KILL 200 $R --master-port 29981 scripts/dbg_stage_n4.py 2>&1 | grep -E "status|Error" | head -40
DBG_T=1024 timeout -s KILL 200 $R --master-port 29982 scripts/dbg_stage_n4.py 2>&1 | grep -E "status|Error" | head -10
exit 0
