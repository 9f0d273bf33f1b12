#!/usr/bin/env python
"""Same-box A/B of the expert FFN between two builds of libmsinfer.so (only
msi_pack_w13 + msi_grouped_ffn are bound, so an older build works too).
usage: ab_lib_ffn.py LIB_A LIB_B [rounds]  -> median ms per shape and build."""

import ctypes
import json
import statistics
import sys

import torch

P, I = ctypes.c_void_p, ctypes.c_int


def bind(path):
    lib = ctypes.CDLL(path)
    lib.msi_pack_w13.argtypes = [P, P, P, I, I, I, P]
    lib.msi_grouped_ffn.argtypes = [P, P, I, I, P, P, P, P, I, I, P]
    return lib


def main():
    libs = [bind(p) for p in sys.argv[1:3]]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    H, Hp = 6144, 16384
    torch.manual_seed(0)
    res = {}
    for E_l, per in ((8, 768), (4, 1536)):
        cnt = [per + 37 * ((e * 5) % 7 - 3) for e in range(E_l)]
        starts, run = [], 0
        for c in cnt:
            starts.append(run)
            run += (c + 127) // 128 * 128
        rows = run
        x = torch.randn(rows, H, device="cuda").to(torch.bfloat16)
        gate = (torch.randn(E_l, Hp, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
        up = (torch.randn(E_l, Hp, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
        w2 = (torch.randn(E_l, H, Hp, device="cuda") / Hp ** 0.5).to(torch.bfloat16)
        tot = torch.tensor(cnt, dtype=torch.int32, device="cuda")
        hbuf = torch.empty(rows, Hp, dtype=torch.bfloat16, device="cuda")
        ys = []
        for k, lib in enumerate(libs):
            w13 = torch.empty(E_l, 2 * Hp, H, dtype=torch.bfloat16, device="cuda")
            s = torch.cuda.current_stream().cuda_stream
            assert lib.msi_pack_w13(gate.data_ptr(), up.data_ptr(), w13.data_ptr(), E_l, Hp, H, s) == 0
            ys.append((lib, w13, torch.zeros(rows, H, dtype=torch.bfloat16, device="cuda")))
        times = [[] for _ in libs]
        for r in range(rounds * 4):
            for k, (lib, w13, y) in enumerate(ys):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s = torch.cuda.current_stream().cuda_stream
                a.record()
                assert lib.msi_grouped_ffn(x.data_ptr(), tot.data_ptr(), E_l, rows, w13.data_ptr(), w2.data_ptr(),
                                           hbuf.data_ptr(), y.data_ptr(), H, Hp, s) == 0
                b.record()
                torch.cuda.synchronize()
                if r >= 2:
                    times[k].append(a.elapsed_time(b))
        same = torch.equal(ys[0][2], ys[1][2])
        fl = 6.0 * sum(cnt) * H * Hp
        res[f"E{E_l}x{per}"] = {"ms": [statistics.median(t) for t in times],
                                "tflops": [fl / statistics.median(t) / 1e9 for t in times], "bit_identical": same}
    print(json.dumps({"libs": sys.argv[1:3], **res}))


if __name__ == "__main__":
    main()
