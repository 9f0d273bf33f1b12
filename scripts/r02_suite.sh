#!/bin/bash
# full GPU suite + smoke on one GPU (what the driver runs), FFN determinism
set -u
mkdir -p gpurun_out
timeout 300 python scripts/det_ffn.py
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_full.log 2>&1; tail -5 gpurun_out/r02_pytest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
