#!/bin/bash
# full GPU suite on a 4-GPU box (multi-rank tests on real NVLink peers) + smoke
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke4.log 2>&1; tail -1 gpurun_out/smoke4.log
