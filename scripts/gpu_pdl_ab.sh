#!/bin/bash
# PDL A/B (gpurun --gpus 2): GPU tests with MSI_PDL=1, then M2N round trips
# (1+1 and co-located, eager / graph / chained) and the N=1 bench with PDL off / on.
set -u
mkdir -p gpurun_out
MSI_PDL=1 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_pdl.log 2>&1; tail -2 gpurun_out/pytest_pdl.log
for P in 0 1; do
  for C in "" "--colocated"; do
    MSI_PDL=$P timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2952$P \
      bench_m2n.py $C --shape mixtral-8x22b --sizes 1,16,128,1024,3072 --iters 400 --chain 16 > gpurun_out/m2n_pdl${P}${C}.log 2>&1
    grep '^{' gpurun_out/m2n_pdl${P}${C}.log > gpurun_out/m2n_pdl${P}${C}.jsonl
  done
done
for P in 0 1 0 1; do
  MSI_PDL=$P timeout 300 python bench.py --no-cpu --no-e2e --no-m2n --steps 20 > gpurun_out/bench_pdl$P.log 2>&1
  grep '^{' gpurun_out/bench_pdl$P.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('PDL', $P, d['value'], d['clocks']['sm_mhz'])"
done
