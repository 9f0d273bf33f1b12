#!/bin/bash
# NVLink byte counters of the M2N kernels, co-located 2 GPUs, one pass (no replay), gloo host collectives
set -u
mkdir -p gpurun_out
export MSI_M2N_BACKEND=gloo
timeout -s KILL 300 ncu --target-processes all --graph-profiling node --clock-control none \
  --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k "regex:dispatch" -c 8 --csv \
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
  bench_m2n.py --colocated --shape mixtral-8x22b --sizes 3072 --iters 3 --warmup 1 --no-nccl --chain 1 \
  > gpurun_out/r02_ncu_nvl_n2_disp.csv 2> gpurun_out/r02_ncu_nvl_n2_disp.err
echo "rc=$?"; grep -c nvltx gpurun_out/r02_ncu_nvl_n2_disp.csv; grep -E "nvltx|nvlrx" gpurun_out/r02_ncu_nvl_n2_disp.csv | head -8 | cut -c1-300
