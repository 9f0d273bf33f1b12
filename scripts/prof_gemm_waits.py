#!/usr/bin/env python
"""Where does the expert GEMM's MMA issuer wait?  Runs msi_grouped_ffn at the
N = 1 headline shape (Mixtral-8x22B, 8 experts x ~768 rows) with a build made
with -DMSI_GEMM_PROF=1 and prints, summed over all CTA-pair leaders of both
GEMMs: the fraction of the issuer loop spent waiting for operand stages (TMA
not ahead), waiting for a free TMEM accumulator (epilogue not done), and the
average cycles per tile.
usage: prof_gemm_waits.py LIB_WITH_PROF [E_l per]"""

import ctypes
import json
import sys

import torch

P, I = ctypes.c_void_p, ctypes.c_int


def main():
    lib = ctypes.CDLL(sys.argv[1])
    lib.msi_pack_w13.argtypes = [P, P, P, I, I, I, P]
    lib.msi_grouped_ffn.argtypes = [P, P, I, I, P, P, P, P, I, I, P]
    lib.msi_dbg_gemm_prof.argtypes = [P]
    E_l = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    per = int(sys.argv[3]) if len(sys.argv) > 3 else 768
    H, Hp = 6144, 16384
    torch.manual_seed(0)
    cnt = [per + 37 * ((e * 5) % 7 - 3) for e in range(E_l)]
    rows = sum((c + 127) // 128 * 128 for c in cnt)
    x = torch.randn(rows, H, device="cuda").to(torch.bfloat16)
    gate = (torch.randn(E_l, Hp, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
    up = (torch.randn(E_l, Hp, H, device="cuda") / H ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn(E_l, H, Hp, device="cuda") / Hp ** 0.5).to(torch.bfloat16)
    tot = torch.tensor(cnt, dtype=torch.int32, device="cuda")
    hbuf = torch.empty(rows, Hp, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(rows, H, dtype=torch.bfloat16, device="cuda")
    w13 = torch.empty(E_l, 2 * Hp, H, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert lib.msi_pack_w13(gate.data_ptr(), up.data_ptr(), w13.data_ptr(), E_l, Hp, H, s) == 0
    prof = (ctypes.c_ulonglong * 4)()

    def ffn():
        assert lib.msi_grouped_ffn(x.data_ptr(), tot.data_ptr(), E_l, rows, w13.data_ptr(), w2.data_ptr(),
                                   hbuf.data_ptr(), y.data_ptr(), H, Hp, s) == 0

    for _ in range(4):
        ffn()
    torch.cuda.synchronize()
    lib.msi_dbg_gemm_prof(prof)
    n = 8
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        ffn()
    b.record()
    torch.cuda.synchronize()
    assert lib.msi_dbg_gemm_prof(prof) == 0
    w_full, w_acc, loop, tiles = list(prof)
    ms = a.elapsed_time(b) / n
    print(json.dumps({"E_l": E_l, "per": per, "ffn_ms": round(ms, 3),
                      "tflops": round(6.0 * sum(cnt) * H * Hp / ms / 1e9, 1),
                      "wait_operands_frac": round(w_full / loop, 4), "wait_accumulator_frac": round(w_acc / loop, 4),
                      "cycles_per_tile": round(loop / tiles), "tiles_per_call": tiles // n}))


if __name__ == "__main__":
    main()
