#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "router or regression" 2>&1 | tail -2
timeout 300 python scripts/ab_route_tiles.py 2>/dev/null
timeout 300 python scripts/ab_router_tc.py 2>/dev/null
