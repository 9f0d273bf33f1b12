#!/bin/bash
# final code: the driver's bench commands at N=1, 2, 4 (one 4-GPU box) + the reference arm at N=1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/fb_n1.log 2>&1; echo "n1 rc=$?"; grep '^{' gpurun_out/fb_n1.log | tail -1 > gpurun_out/fb_n1.json
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --gpus $n > gpurun_out/fb_n$n.log 2>&1; echo "n$n rc=$?"
  grep '^{' gpurun_out/fb_n$n.log | tail -1 > gpurun_out/fb_n$n.json
done
timeout 900 python bench.py --impl reference > gpurun_out/fb_ref.log 2>&1; echo "ref rc=$?"; grep '^{' gpurun_out/fb_ref.log | tail -1 > gpurun_out/fb_ref.json
