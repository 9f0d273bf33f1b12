#!/bin/bash
# Final single-GPU pass of a round (gpurun, 1 GPU): the full GPU test suite and
# smoke, then scripts/profile_n1.sh (bench line, launch list, ncu --set full of
# GEMM1/GEMM2 and decode attention), then ncu tensor-pipe metrics of the expert
# GEMM at the per-GPU shapes of the co-located N = 2 and N = 4 layouts
# (4 local experts x t_e 1536, 2 local experts x t_e 3072).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
bash scripts/profile_n1.sh > gpurun_out/profile_n1.log 2>&1; tail -3 gpurun_out/profile_n1.log
NCU=/usr/local/cuda/bin/ncu
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed"
for cfg in "4 1536" "2 3072"; do
  set -- $cfg
  timeout 600 python bench_gemm.py --experts $1 --te $2 --iters 3 > gpurun_out/gemm_e$1_t$2.log 2>&1
  timeout 900 $NCU --metrics $M --clock-control none --csv -k regex:grouped_gemm -s 4 -c 2 \
      python bench_gemm.py --experts $1 --te $2 --iters 1 > gpurun_out/ncu_gemm_e$1_t$2.csv 2>&1 || echo "ncu e$1 t$2 failed"
done
ls gpurun_out
