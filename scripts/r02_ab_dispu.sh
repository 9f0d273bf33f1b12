#!/bin/bash
# dispatch copy unroll A/B: default build (U=8) vs U=12 vs U=24, same box, route_dispatch at the N=1 shape
cp paper_2504_02263_b200/libmsinfer.so /tmp/lib_u8.so
for rep in 1 2; do
  for u in 8 12 24; do
    if [ $u = 8 ]; then cp /tmp/lib_u8.so paper_2504_02263_b200/libmsinfer.so; else cp scripts/ab_libs/libmsinfer_u$u.so paper_2504_02263_b200/libmsinfer.so; fi
    echo "U=$u $(timeout 120 python scripts/ab_route_tiles.py 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["route_dispatch_us"]["default"], d["route_dispatch_us"]["4x8x24"])')"
  done
done
cp /tmp/lib_u8.so paper_2504_02263_b200/libmsinfer.so
