#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 python scripts/ab_l2hint.py
timeout 300 python scripts/ab_l2hint.py
cat > /tmp/ffn_one.py <<'PY'
import os, sys, torch
sys.path.insert(0, '.')
from paper_2504_02263_b200 import ops, runtime
from paper_2504_02263_b200.config import as_model_spec
m = as_model_spec("mixtral-8x22b"); E_l, per = 8, 768
cnt = [per + 37 * ((e * 5) % 7 - 3) for e in range(E_l)]
st = ops.segment_starts(cnt); rows = st[-1] + (cnt[-1] + 127) // 128 * 128
_, w13, w2 = runtime.synth_device_weights(m, list(range(E_l)), seed=0, device="cuda")
x = torch.randn(rows, m.hidden, device="cuda").to(torch.bfloat16)
tot = torch.tensor(cnt, dtype=torch.int32, device="cuda")
for _ in range(2): ops.grouped_ffn(x, tot, w13, w2)
torch.cuda.synchronize()
PY
for h in 0 1; do
  MSI_GEMM_L2HINT=$h timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:grouped_gemm -s 2 -c 2 --csv python /tmp/ffn_one.py 2>/dev/null | grep -E "dram__bytes|time_dur|tensor" | awk -F'","' -v h=$h '{print "hint=" h, $(NF-2), $NF}'
done
