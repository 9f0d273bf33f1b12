#!/usr/bin/env python
"""Same-box A/B of the DeepSeek-V3-shaped router (E = 256, K = 8, h = 7168)
between builds of libmsinfer.so and tensor-core tile sizes (MSI_ROUTER_TC_BT).
Each timing is 20 back-to-back msi_gate_topk calls between two CUDA events
(the GPU stays ahead of the host), median of 7; outputs must be bit-identical
to the pinned-order CUDA-core path (MSI_ROUTER_TC=0) of the first build.
usage: ab_router_lib.py LIB [LIB ...]   (variants: MSI_AB_BT="8,12,16")"""

import ctypes
import json
import os
import statistics
import sys

import torch

P, I = ctypes.c_void_p, ctypes.c_int


def bind(path):
    lib = ctypes.CDLL(path)
    lib.msi_gate_topk_workspace.restype = ctypes.c_size_t
    lib.msi_gate_topk_workspace.argtypes = [I, I]
    lib.msi_gate_topk.argtypes = [P, P, I, I, I, I, P, P, P, P, P, P]
    lib.msi_gate_topk.restype = I
    return lib


def run(lib, x, wg, K, outs, ws):
    T, H = x.shape
    E = wg.shape[0]
    idx, w, cnt, slot = outs
    rc = lib.msi_gate_topk(x.data_ptr(), wg.data_ptr(), T, H, E, K, idx.data_ptr(), w.data_ptr(),
                           cnt.data_ptr(), slot.data_ptr(), ws.data_ptr(),
                           torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc


def main():
    libs = [(os.path.basename(p), bind(p)) for p in sys.argv[1:]]
    bts = [int(b) for b in os.environ.get("MSI_AB_BT", "0").split(",")]
    H, E, K = 7168, 256, 8
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    wg = (torch.randn(E, H, generator=g, device="cuda") / H ** 0.5).to(torch.bfloat16)
    for T in [int(t) for t in os.environ.get("MSI_AB_T", "1024,2048,4096").split(",")]:
        x = torch.randn(T, H, generator=g, device="cuda").to(torch.bfloat16)
        ws = torch.zeros(libs[0][1].msi_gate_topk_workspace(T, E), dtype=torch.uint8, device="cuda")

        def new_outs():
            return (torch.empty((T, K), dtype=torch.int32, device="cuda"),
                    torch.empty((T, K), dtype=torch.float32, device="cuda"),
                    torch.empty((E,), dtype=torch.int32, device="cuda"),
                    torch.empty((T, K), dtype=torch.int32, device="cuda"))

        os.environ["MSI_ROUTER_TC"] = "0"
        ref = new_outs()
        run(libs[0][1], x, wg, K, ref, ws)
        res = {"T": T}
        ts, o0 = [], new_outs()
        for _ in range(7):  # the pinned-order CUDA-core path, last build
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                run(libs[-1][1], x, wg, K, o0, ws)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / 20)
        res["pinned_cuda_core_us"] = round(statistics.median(ts), 1)
        os.environ["MSI_ROUTER_TC"] = "1"
        for name, lib in libs:
            for bt in bts:
                if bt:
                    os.environ["MSI_ROUTER_TC_BT"] = str(bt)
                else:
                    os.environ.pop("MSI_ROUTER_TC_BT", None)
                o = new_outs()
                ts = []
                for _ in range(7):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(20):
                        run(lib, x, wg, K, o, ws)
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b) * 1e3 / 20)
                key = f"{name}|bt{bt or 'default'}"
                res[key + "_us"] = round(statistics.median(ts), 1)
                res[key + "_identical"] = all(torch.equal(u, v) for u, v in zip(o, ref))
        os.environ.pop("MSI_ROUTER_TC_BT", None)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
