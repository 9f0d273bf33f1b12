#!/bin/bash
cp paper_2504_02263_b200/libmsinfer.so /tmp/lib_new.so
for rep in 1 2 3; do
  for v in prev new; do
    if [ $v = new ]; then cp /tmp/lib_new.so paper_2504_02263_b200/libmsinfer.so; else cp scripts/ab_libs/libmsinfer_prevhead.so paper_2504_02263_b200/libmsinfer.so; fi
    echo "$v $(timeout 120 python scripts/ab_route_tiles.py 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["route_dispatch_us"]["default"])')"
  done
done
cp /tmp/lib_new.so paper_2504_02263_b200/libmsinfer.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k router 2>&1 | tail -1
