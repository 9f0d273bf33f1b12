#!/bin/bash
# combine kernel: resident CTAs per SM (grid = m x SMs), ncu per-launch durations at the N=1 bench step
mkdir -p gpurun_out
SMALL="--steps 1 --warmup 3 --no-e2e --no-cpu --no-graph --no-m2n"
for m in 4 6 8 4; do
  MSI_COMBINE_CTAS=$m timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:combine \
     python bench.py $SMALL 2>/dev/null | grep combine_kernel | python -c "
import sys, csv
rows = list(csv.reader(sys.stdin))
t = [float(r[-1].replace(',', '')) for r in rows if r[-3] == 'gpu__time_duration.sum']
print('ctas_per_sm=$m', 'launches', len(t), 'median_us', sorted(t)[len(t)//2] / (1e3 if rows and 'nsecond' in rows[0] else 1))
"
done 2>&1 | tee gpurun_out/ab_combine.txt
