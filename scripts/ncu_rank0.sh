#!/bin/bash
# torchrun --no-python scripts/ncu_rank0.sh <python args>: rank 0 runs under ncu
# (one GPU's kernels; the peer rank runs plain), every other rank plain python.
if [ "${LOCAL_RANK:-0}" = "0" ]; then
  exec ncu ${NCU_ARGS:---section SpeedOfLight --section Nvlink} --clock-control none -k "${NCU_K:-regex:.}" -c "${NCU_C:-20}" \
       -o "${NCU_OUT:-gpurun_out/ncu_rank0}" -f python "$@"
fi
exec python "$@"
