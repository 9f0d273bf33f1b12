#!/bin/bash
# r02: host probe + full GPU suite (multi-rank tests share the one GPU)
set -x
(nproc; free -g; lscpu | grep -E "Model name|Flags|Socket|Thread|Core"; nvidia-smi -L) > gpurun_out/r02_host.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu.log 2>&1; tail -3 gpurun_out/r02_pytest_gpu.log
