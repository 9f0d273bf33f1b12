"""Stateless building blocks of the decode step on torch CUDA tensors.

Each function is a thin wrapper over one libmsinfer entry point
(include/msinfer.h); tensors are passed by data pointer on the current torch
stream.  No CPU or PyTorch fallback exists: on a non-B200 device or without
the built library every call raises ``MsiError``.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib

ROW_ALIGN = _lib.ROW_ALIGN


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _check_bf16(name, t, ndim=None):
    if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous CUDA bfloat16 tensor")
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"{name}: expected {ndim} dims, got {tuple(t.shape)}")


class RouterWorkspace:
    """Zero-initialised scratch for gate_topk (the kernel leaves it zeroed)."""

    def __init__(self, max_tokens: int, experts: int, device=None):
        n = _lib.load().msi_gate_topk_workspace(max_tokens, experts)
        self.buf = torch.zeros(n, dtype=torch.uint8, device=device or "cuda")
        self.max_tokens = max_tokens


def gate_topk(x: torch.Tensor, wg: torch.Tensor, topk: int, ws: RouterWorkspace | None = None,
              out=None, stream=None):
    """Router: -> idx [T,K] i32, w [T,K] f32, cnt [E] i32,
    slot [T,K] i32.  Bit-exact with the oracle."""
    _check_bf16("x", x, 2)
    _check_bf16("wg", wg, 2)
    T, H = x.shape
    E = wg.shape[0]
    if wg.shape[1] != H:
        raise ValueError("wg must be [E, H]")
    if ws is None or ws.max_tokens < T:
        ws = RouterWorkspace(max(T, 1), E, x.device)
    if out is None:
        idx = torch.empty((T, topk), dtype=torch.int32, device=x.device)
        w = torch.empty((T, topk), dtype=torch.float32, device=x.device)
        cnt = torch.empty((E,), dtype=torch.int32, device=x.device)
        slot = torch.empty((T, topk), dtype=torch.int32, device=x.device)
    else:
        idx, w, cnt, slot = out
    _lib.call("msi_gate_topk", _ptr(x), _ptr(wg), T, H, E, topk, _ptr(idx), _ptr(w), _ptr(cnt),
              _ptr(slot), _ptr(ws.buf), _stream(stream))
    return idx, w, cnt, slot


def pack_w13(w_gate: torch.Tensor, w_up: torch.Tensor, stream=None) -> torch.Tensor:
    """[E_l, H', H] gate + up -> [E_l, 2H', H]: each 256-row GEMM1 N tile holds
    [gate 64 | up 64 | gate 64 | up 64] of 128 consecutive features."""
    _check_bf16("w_gate", w_gate, 3)
    _check_bf16("w_up", w_up, 3)
    E_l, Hp, H = w_gate.shape
    out = torch.empty((E_l, 2 * Hp, H), dtype=torch.bfloat16, device=w_gate.device)
    _lib.call("msi_pack_w13", _ptr(w_gate), _ptr(w_up), _ptr(out), E_l, Hp, H, _stream(stream))
    return out


def segment_starts(total) -> list[int]:
    starts, run = [], 0
    for t in total:
        starts.append(run)
        run += (int(t) + ROW_ALIGN - 1) // ROW_ALIGN * ROW_ALIGN
    return starts


def grouped_ffn(x_rows: torch.Tensor, total: torch.Tensor, w13: torch.Tensor, w2: torch.Tensor,
                hbuf: torch.Tensor | None = None, y: torch.Tensor | None = None, stream=None):
    """Grouped SwiGLU FFN on the tcgen05 GEMM.  x_rows [rows, H] laid out in
    128-row aligned per-expert segments (``segment_starts``); total [E_l] int32
    on device.  Returns y [rows, H] (rows beyond each segment are untouched)."""
    _check_bf16("x_rows", x_rows, 2)
    rows, H = x_rows.shape
    E_l, two_hp, _ = w13.shape
    Hp = two_hp // 2
    if hbuf is None:
        hbuf = torch.empty((rows, Hp), dtype=torch.bfloat16, device=x_rows.device)
    if y is None:
        y = torch.zeros((rows, H), dtype=torch.bfloat16, device=x_rows.device)
    total = total.to(device=x_rows.device, dtype=torch.int32).contiguous()
    _lib.call("msi_grouped_ffn", _ptr(x_rows), _ptr(total), E_l, rows, _ptr(w13), _ptr(w2),
              _ptr(hbuf), _ptr(y), H, Hp, _stream(stream))
    return y


def combine_local(y: torch.Tensor, w: torch.Tensor, resid: torch.Tensor | None = None,
                  out: torch.Tensor | None = None, stream=None):
    """out[t] = bf16(resid[t] + sum_k w[t,k] y[t,k])."""
    _check_bf16("y", y, 3)
    T, K, H = y.shape
    if out is None:
        out = torch.empty((T, H), dtype=torch.bfloat16, device=y.device)
    _lib.call("msi_combine_local", _ptr(y), _ptr(w.contiguous()), _ptr(resid), _ptr(out), T, K, H,
              _stream(stream))
    return out


# ---------------------------------------------------------- attention ---- #
def _check_i32(name, t):
    if t.dtype != torch.int32 or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous CUDA int32 tensor")


def rope_append(qkv: torch.Tensor, pos: torch.Tensor, n_heads: int, n_kv: int, theta: float,
                block_table: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor,
                q_out: torch.Tensor, stream=None) -> torch.Tensor:
    """RoPE on the new token's q, k at ``pos`` + KV append (msi_rope_append).
    qkv bf16 [T, >= (n_heads + 2 n_kv) 128] (row stride may exceed the width);
    caches bf16 [pages, n_kv, 64, 128]; q_out bf16 [T, n_heads, 128]."""
    if qkv.dtype != torch.bfloat16 or not qkv.is_cuda or qkv.stride(1) != 1:
        raise ValueError("rope_append: qkv must be a row-major CUDA bfloat16 matrix")
    _check_i32("pos", pos)
    _check_i32("block_table", block_table)
    for n, t in (("k_cache", k_cache), ("v_cache", v_cache), ("q_out", q_out)):
        _check_bf16(n, t)
    _lib.call("msi_rope_append", _ptr(qkv), qkv.stride(0), _ptr(pos), qkv.shape[0], n_heads, n_kv,
              ctypes.c_float(theta), _ptr(block_table), block_table.shape[1], _ptr(k_cache), _ptr(v_cache),
              k_cache.shape[0], _ptr(q_out), _stream(stream))
    return q_out


def decode_attention_workspace(T: int, n_heads: int, n_kv: int, max_pages: int, device=None) -> torch.Tensor | None:
    n = _lib.load().msi_decode_attention_workspace(T, n_heads, n_kv, max_pages)
    return torch.empty(n, dtype=torch.uint8, device=device) if n else None


def decode_attention(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, block_table: torch.Tensor,
                     seq_lens: torch.Tensor, out: torch.Tensor, workspace: torch.Tensor | None = None,
                     scale: float | None = None, stream=None) -> torch.Tensor:
    """GQA decode attention over the paged cache (msi_decode_attention).
    q bf16 [T, n_heads, 128]; out bf16 [T, n_heads * 128]."""
    for n, t in (("q", q), ("k_cache", k_cache), ("v_cache", v_cache), ("out", out)):
        _check_bf16(n, t)
    _check_i32("block_table", block_table)
    _check_i32("seq_lens", seq_lens)
    T, n_heads, d = q.shape
    n_kv = k_cache.shape[1]
    if k_cache.shape[2:] != (_lib.KV_PAGE, _lib.HEAD_DIM) or d != _lib.HEAD_DIM:
        raise ValueError("decode_attention: caches must be [pages, n_kv, 64, 128], q [T, heads, 128]")
    if workspace is None:
        workspace = decode_attention_workspace(T, n_heads, n_kv, block_table.shape[1], q.device)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    scale = d ** -0.5 if scale is None else scale
    _lib.call("msi_decode_attention", _ptr(q), _ptr(k_cache), _ptr(v_cache), k_cache.shape[0], _ptr(block_table),
              block_table.shape[1], _ptr(seq_lens), T, n_heads, n_kv, ctypes.c_float(scale), _ptr(out),
              _ptr(workspace), ws_bytes, _stream(stream))
    return out


class TileCounter:
    """Zeroed device words for the dense GEMM launches' dynamic tile
    scheduler (each launch leaves its word at 0; one in-flight launch per word)."""

    def __init__(self, n: int = 1, device=None):
        self.buf = torch.zeros(n * 32, dtype=torch.int32, device=device or "cuda")  # 128 B apart

    def __getitem__(self, i: int):
        return ctypes.c_void_p(self.buf.data_ptr() + 128 * i)


def dense_gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None,
               resid: torch.Tensor | None = None, ctr: TileCounter | None = None, slot: int = 0,
               stream=None) -> torch.Tensor:
    """out = bf16(a b^T (+ resid)) on the tcgen05 GEMM (msi_dense_gemm):
    a bf16 [T, K], b bf16 [N, K]; out/resid bf16 [T, >= N] row-major."""
    _check_bf16("a", a, 2)
    _check_bf16("b", b, 2)
    T, K = a.shape
    N = b.shape[0]
    if b.shape[1] != K:
        raise ValueError("dense_gemm: b must be [N, K]")
    if out is None:
        out = torch.empty((T, N), dtype=torch.bfloat16, device=a.device)
    for name, t in (("out", out), ("resid", resid)):
        if t is not None and (t.dtype != torch.bfloat16 or not t.is_cuda or t.stride(1) != 1 or t.shape[0] != T):
            raise ValueError(f"dense_gemm: {name} must be a row-major CUDA bfloat16 [T, >= N] matrix")
    ctr = ctr or TileCounter(1, a.device)
    _lib.call("msi_dense_gemm", _ptr(a), T, _ptr(b), N, K, _ptr(out), out.stride(0), _ptr(resid),
              0 if resid is None else resid.stride(0), ctr[slot], _stream(stream))
    return out


def qkv_rope_append(x: torch.Tensor, wqkv: torch.Tensor, pos: torch.Tensor, n_heads: int, n_kv: int,
                    theta: float, block_table: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor,
                    q_out: torch.Tensor, ctr: TileCounter | None = None, slot: int = 0, stream=None) -> torch.Tensor:
    """QKV projection with RoPE + paged-KV append in the GEMM epilogue
    (msi_qkv_rope_append): the result msi_rope_append gives on bf16(x wqkv^T)."""
    _check_bf16("x", x, 2)
    _check_bf16("wqkv", wqkv, 2)
    _check_i32("pos", pos)
    _check_i32("block_table", block_table)
    for n, t in (("k_cache", k_cache), ("v_cache", v_cache), ("q_out", q_out)):
        _check_bf16(n, t)
    T, H = x.shape
    if wqkv.shape != ((n_heads + 2 * n_kv) * _lib.HEAD_DIM, H):
        raise ValueError("qkv_rope_append: wqkv must be [(n_heads + 2 n_kv) 128, hidden]")
    ctr = ctr or TileCounter(1, x.device)
    _lib.call("msi_qkv_rope_append", _ptr(x), T, H, _ptr(wqkv), n_heads, n_kv, _ptr(pos), ctypes.c_float(theta),
              _ptr(block_table), block_table.shape[1], _ptr(k_cache), _ptr(v_cache), _ptr(q_out), ctr[slot],
              _stream(stream))
    return q_out


def grouped_ffn_regions(x_reg: torch.Tensor, counts, cap_s: int, w13: torch.Tensor, w2: torch.Tensor,
                        y_reg: torch.Tensor | None = None, hbuf: torch.Tensor | None = None, a_runs: bool = True,
                        gather: bool = False, stream=None) -> torch.Tensor:
    """The expert FFN on (expert, sender) receive regions (msi_grouped_ffn_regions):
    x_reg bf16 [E_l * n_src * cap_s, H], region (e, s) = rows
    [(e n_src + s) cap_s, + counts[s][e]).  Returns y_reg (Y of each row at
    its own row; may be x_reg itself).  gather=True: regions gathered into
    compact per-expert segments first (msi_expert_ffn with several senders)."""
    _check_bf16("x_reg", x_reg, 2)
    E_l, two_hp, H = w13.shape
    Hp = two_hp // 2
    cnt = torch.as_tensor(counts, dtype=torch.int64)
    n_src = cnt.shape[0]
    if cnt.shape != (n_src, E_l) or x_reg.shape[0] < E_l * n_src * cap_s or (cnt > cap_s).any():
        raise ValueError("grouped_ffn_regions: counts must be [n_src, E_l] <= cap_s over E_l*n_src*cap_s rows")
    tab = cnt.to(x_reg.device).contiguous()
    tot = cnt.sum(0).tolist()
    rows = sum((int(t) + ROW_ALIGN - 1) // ROW_ALIGN * ROW_ALIGN for t in tot) + ROW_ALIGN
    if hbuf is None:
        hbuf = torch.empty((rows, Hp), dtype=torch.bfloat16, device=x_reg.device)
    if y_reg is None:
        y_reg = torch.zeros_like(x_reg)
    xcomp = torch.empty((hbuf.shape[0], H), dtype=torch.bfloat16, device=x_reg.device) if gather else None
    _lib.call("msi_grouped_ffn_regions", _ptr(x_reg), _ptr(tab), n_src, cap_s, E_l, _ptr(w13), _ptr(w2),
              _ptr(hbuf), hbuf.shape[0], _ptr(y_reg), H, Hp, int(a_runs), _ptr(xcomp), _stream(stream))
    return y_reg


def dense_logits(x: torch.Tensor, wg: torch.Tensor, ctr: TileCounter | None = None, stream=None) -> torch.Tensor:
    """fp32 x wg^T on the tensor cores (msi_dense_logits; E % 256 == 0)."""
    _check_bf16("x", x, 2)
    _check_bf16("wg", wg, 2)
    out = torch.empty((x.shape[0], wg.shape[0]), dtype=torch.float32, device=x.device)
    ctr = ctr or TileCounter(1, x.device)
    _lib.call("msi_dense_logits", _ptr(x), x.shape[0], _ptr(wg), wg.shape[0], wg.shape[1], _ptr(out), ctr[0],
              _stream(stream))
    return out
