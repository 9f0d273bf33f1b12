#!/usr/bin/env python
"""Same-process A/B of TMA L2 eviction hints (MSI_GEMM_L2HINT) on the expert
FFN at the N = 1 / N = 2 shapes; interleaved, medians."""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_02263_b200 import ops, runtime  # noqa: E402
from paper_2504_02263_b200.config import as_model_spec  # noqa: E402


def main():
    model = as_model_spec("mixtral-8x22b")
    H, Hp = model.hidden, model.intermediate
    out = {}
    for E_l, per in ((8, 768), (4, 1536)):
        cnt = [per + 37 * ((e * 5) % 7 - 3) for e in range(E_l)]
        starts = ops.segment_starts(cnt)
        rows = starts[-1] + (cnt[-1] + 127) // 128 * 128
        _, w13, w2 = runtime.synth_device_weights(model, list(range(E_l)), seed=0, device="cuda")
        x = torch.randn(rows, H, device="cuda").to(torch.bfloat16)
        tot = torch.tensor(cnt, dtype=torch.int32, device="cuda")
        hb = torch.empty(rows, Hp, dtype=torch.bfloat16, device="cuda")
        y = torch.empty(rows, H, dtype=torch.bfloat16, device="cuda")
        ts = {"0": [], "1": []}
        ys = {}
        for r in range(16):
            for mode in ("0", "1"):
                os.environ["MSI_GEMM_L2HINT"] = mode
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                ops.grouped_ffn(x, tot, w13, w2, hb, y)
                b.record()
                torch.cuda.synchronize()
                if r >= 2:
                    ts[mode].append(a.elapsed_time(b))
                ys[mode] = y.clone()
        fl = 6.0 * sum(cnt) * H * Hp
        out[f"E{E_l}x{per}"] = {m: {"ms": statistics.median(v), "tflops": fl / statistics.median(v) / 1e9}
                                for m, v in ts.items()}
        out[f"E{E_l}x{per}"]["bit_identical"] = torch.equal(ys["0"], ys["1"])
        del w13, w2
    print(json.dumps(out))


if __name__ == "__main__":
    main()
