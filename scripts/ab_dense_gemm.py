#!/usr/bin/env python
"""Attention projections: msi_dense_gemm / msi_qkv_rope_append (tcgen05) vs
cuBLAS (torch.matmul / addmm) at the bench shapes; medians of CUDA-event times."""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_02263_b200 import _lib, ops  # noqa: E402
from paper_2504_02263_b200 import attention as A  # noqa: E402
from paper_2504_02263_b200.config import as_model_spec  # noqa: E402


def timeit(fn, iters=20):
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts[3:])


def main():
    model = as_model_spec(os.environ.get("AB_SHAPE", "mixtral-8x22b"))
    out = []
    for T in [int(v) for v in os.environ.get("AB_T", "3072,1024,256").split(",")]:
        st = A.AttentionStage(model, T, 1, "cuda", seed=1)
        x = torch.randn(T, model.hidden, device="cuda").to(torch.bfloat16)
        c = st.cache
        qkv = torch.empty(T, st.qkv_width, dtype=torch.bfloat16, device="cuda")
        y = torch.empty(T, model.hidden, dtype=torch.bfloat16, device="cuda")
        ctr = ops.TileCounter(2)
        r = {"T": T, "shape": model.name}
        flq = 2.0 * T * model.hidden * st.qkv_width
        flo = 2.0 * T * model.hidden * st.o.shape[1]
        for cg in (2, 1):
            _lib.call("msi_set_gemm_cta_group", cg)
            r[f"qkv_dense_cg{cg}_us"] = timeit(lambda: ops.dense_gemm(x, st.w.wqkv, qkv, ctr=ctr))
            r[f"qkv_rope_cg{cg}_us"] = timeit(lambda: ops.qkv_rope_append(x, st.w.wqkv, c.pos, st.n_heads, st.n_kv,
                                                                          st.theta, c.block_table, c.k[0], c.v[0],
                                                                          st.q, ctr))
            r[f"oproj_cg{cg}_us"] = timeit(lambda: ops.dense_gemm(st.o, st.w.wo, y, resid=x, ctr=ctr, slot=1))
        _lib.call("msi_set_gemm_cta_group", 0)
        r["qkv_cublas_us"] = timeit(lambda: torch.matmul(x, st.w.wqkv.t(), out=qkv))
        r["rope_append_us"] = timeit(lambda: ops.rope_append(qkv, c.pos, st.n_heads, st.n_kv, st.theta,
                                                             c.block_table, c.k[0], c.v[0], st.q))
        r["oproj_cublas_us"] = timeit(lambda: torch.addmm(x, st.o, st.w.wo.t(), out=y))
        r["qkv_tflops_cublas"] = flq / r["qkv_cublas_us"] / 1e6
        r["qkv_tflops_dense_cg2"] = flq / r["qkv_dense_cg2_us"] / 1e6
        r["oproj_tflops_cublas"] = flo / r["oproj_cublas_us"] / 1e6
        r["oproj_tflops_cg2"] = flo / r["oproj_cg2_us"] / 1e6
        out.append(r)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
