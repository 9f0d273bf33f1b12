"""The attention stage on attention GPUs.

The reference treats attention as a timing model only -- T_a = k1 b_a + k2
with k1 proportional to the KV bytes read, 2 b s h bytes / g
(Table 3 GEMMs: QKV projection
h -> h(1 + 2/g), output projection h -> h).  Here it is a real decode layer:

    q, k = RoPE(x W_qkv^T at pos); append k, v into the paged KV cache
                                          (msi_qkv_rope_append: the tcgen05
                                           GEMM with RoPE + append in its
                                           epilogue, no qkv buffer)
    o = softmax(q K^T / sqrt(128)) V      (msi_decode_attention: paged,
                                           GQA, TMA-streamed, HBM-bound)
    y = x + o W_o^T                       (msi_dense_gemm, residual added in
                                           fp32 in the epilogue)

``y`` is the MoE layer's input (router + M2N dispatch) and its residual.

Head layout: n_heads = h / 128 query heads, G = min(g, n_heads) query heads
per KV head (MoeModelSpec.gqa_group, reduced until it divides n_heads),
n_kv = n_heads / G.  For Mixtral-8x22B: 48 heads, 6 KV heads (h/g = 768),
G = 8, which is exactly the per-token KV width the SPEC's 2 b s h / g counts.

Batch composition: each of the T sequences of a micro-batch holds ``ctx``
cached tokens (synthetic, seeded; default uniform on [1, 2 s - 1] so the
mean is the workload's avg_seq_len s = 730, catalog.py:131) and decodes one
new token at position ctx, attending over ctx + 1 tokens.  Pages are 64
tokens; every sequence's pages are drawn from a shuffled pool, so the block
table is genuinely scattered.  Benchmarks re-decode the same position every
step (stationary work); ``advance()`` moves every sequence on by one token.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib, ops

ROPE_THETA = 1e6  # Mixtral's rope_theta (public config; the reference has none)


def head_layout(model) -> tuple[int, int]:
    """(n_heads, n_kv) for a model spec (see module docstring)."""
    if model.hidden % _lib.HEAD_DIM:
        raise ValueError("hidden must be a multiple of the head dim 128")
    n_heads = model.hidden // _lib.HEAD_DIM
    g = max(1, min(int(getattr(model, "gqa_group", 8)), n_heads, 16))
    while n_heads % g:
        g -= 1
    return n_heads, n_heads // g


def batch_composition(T: int, avg_seq_len: int, seed: int = 0, mode: str = "uniform") -> np.ndarray:
    """Cached context length per sequence: 'uniform' on [1, 2s - 1] (mean s)
    or 'fixed' (all s)."""
    if mode == "fixed":
        return np.full(T, avg_seq_len, np.int32)
    if mode != "uniform":
        raise ValueError("mode must be 'uniform' or 'fixed'")
    rng = np.random.default_rng(seed)
    return rng.integers(1, 2 * avg_seq_len, size=T).astype(np.int32)


class PagedKVCache:
    """Per-layer paged K/V caches [pages, n_kv, 64, 128] bf16 for T sequences,
    one shared block table [T, max_pages] int32 (every layer uses the same
    page ids in its own pool)."""

    def __init__(self, T: int, n_kv: int, ctx_lens: np.ndarray, layers: int, device, seed: int = 0,
                 headroom: int = 0, fill: bool = True):
        P = _lib.KV_PAGE
        ctx = np.asarray(ctx_lens, np.int64)
        if ctx.shape != (T,) or (ctx < 0).any():
            raise ValueError("ctx_lens must be T non-negative lengths")
        need = (ctx + 1 + headroom + P - 1) // P
        self.max_pages = int(need.max()) if T else 1
        self.num_pages = max(int(need.sum()), 1)
        rng = np.random.default_rng(seed + 7919)
        perm = rng.permutation(self.num_pages).astype(np.int32)
        bt = np.zeros((T, self.max_pages), np.int32)
        off = 0
        for t in range(T):
            bt[t, : need[t]] = perm[off: off + need[t]]
            off += need[t]
        self.block_table_host = bt
        self.capacity = (need * P).astype(np.int64)  # tokens each sequence's pages hold
        self.block_table = torch.from_numpy(bt).to(device)
        self.ctx_host = ctx.astype(np.int32)
        self.pos = torch.from_numpy(self.ctx_host.copy()).to(device)        # new token's position
        self.lens = (self.pos + 1).to(torch.int32)                          # tokens attended
        self.T, self.n_kv, self.layers, self.headroom = T, n_kv, layers, headroom
        shape = (self.num_pages, n_kv, P, _lib.HEAD_DIM)
        gen = torch.Generator(device=device)
        gen.manual_seed(seed + 17)
        self.k, self.v = [], []
        for _ in range(layers):
            if fill:
                self.k.append(torch.randn(shape, generator=gen, device=device).to(torch.bfloat16))
                self.v.append(torch.randn(shape, generator=gen, device=device).to(torch.bfloat16))
            else:
                self.k.append(torch.zeros(shape, dtype=torch.bfloat16, device=device))
                self.v.append(torch.zeros(shape, dtype=torch.bfloat16, device=device))

    def bytes_per_layer(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.k[0], self.v[0]))

    def kv_bytes_read(self) -> int:
        """Algorithmic K+V bytes one decode step reads per layer."""
        return int((self.ctx_host.astype(np.int64) + 1).sum()) * self.n_kv * _lib.HEAD_DIM * 2 * 2

    def advance(self):
        """Next decode step: every sequence moves on by one token."""
        if (self.ctx_host.astype(np.int64) + 2 > self.capacity).any():
            raise RuntimeError("paged KV cache: a sequence ran out of pages (raise headroom)")
        self.ctx_host = self.ctx_host + 1
        self.pos += 1
        self.lens += 1


class AttentionWeights:
    """W_qkv [(n_heads + 2 n_kv) 128, h] and W_o [h, n_heads 128], bf16,
    N(0, 1/fan_in) (one set shared by the L_sim layers, like the experts)."""

    def __init__(self, model, device, seed: int = 0):
        self.n_heads, self.n_kv = head_layout(model)
        h = model.hidden
        width = (self.n_heads + 2 * self.n_kv) * _lib.HEAD_DIM
        gen = torch.Generator(device=device)
        gen.manual_seed(seed + 101)
        self.wqkv = (torch.randn((width, h), generator=gen, device=device) / math.sqrt(h)).to(torch.bfloat16)
        self.wo = (torch.randn((h, self.n_heads * _lib.HEAD_DIM), generator=gen, device=device)
                   / math.sqrt(self.n_heads * _lib.HEAD_DIM)).to(torch.bfloat16)


class AttentionStage:
    """One micro-batch's attention stage: T sequences, L layers of KV cache."""

    def __init__(self, model, T: int, layers: int, device, weights: AttentionWeights | None = None,
                 ctx_lens: np.ndarray | None = None, avg_seq_len: int = 730, seed: int = 0,
                 theta: float = ROPE_THETA, composition: str = "uniform", headroom: int = 0):
        self.model, self.T, self.theta = model, T, theta
        self.w = weights or AttentionWeights(model, device, seed)
        self.n_heads, self.n_kv = self.w.n_heads, self.w.n_kv
        if ctx_lens is None:
            ctx_lens = batch_composition(T, avg_seq_len, seed, composition)
        self.cache = PagedKVCache(T, self.n_kv, ctx_lens, layers, device, seed, headroom=headroom)
        D = _lib.HEAD_DIM
        self.qkv_width = (self.n_heads + 2 * self.n_kv) * D
        self.ctr = ops.TileCounter(2, device)  # tile counters of the two projection GEMMs
        self.q = torch.empty((T, self.n_heads, D), dtype=torch.bfloat16, device=device)
        self.o = torch.empty((T, self.n_heads * D), dtype=torch.bfloat16, device=device)
        self.y = torch.empty((T, model.hidden), dtype=torch.bfloat16, device=device)
        self.ws = ops.decode_attention_workspace(T, self.n_heads, self.n_kv, self.cache.max_pages, device)
        self.timing = None  # set to a list to collect attention-kernel events

    def forward(self, x: torch.Tensor, layer: int, out: torch.Tensor | None = None) -> torch.Tensor:
        """x bf16 [T, h] -> x + Attn(x) W_o^T (bf16 [T, h]) on the current stream."""
        c = self.cache
        out = self.y if out is None else out
        ops.qkv_rope_append(x, self.w.wqkv, c.pos, self.n_heads, self.n_kv, self.theta, c.block_table,
                            c.k[layer], c.v[layer], self.q, self.ctr, 0)
        if self.timing is not None:  # (start, end) events around the attention kernel
            e0, e1 = torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True)
            e0.record()
        ops.decode_attention(self.q, c.k[layer], c.v[layer], c.block_table, c.lens, self.o, self.ws)
        if self.timing is not None:
            e1.record()
            self.timing.append((e0, e1))
        ops.dense_gemm(self.o, self.w.wo, out, resid=x, ctr=self.ctr, slot=1)
        return out

    def flops(self) -> float:
        """Projection GEMM FLOPs per layer (Table 3: QKV + output)."""
        h = self.model.hidden
        return 2.0 * self.T * h * (self.qkv_width + self.o.shape[1])

    def attn_bytes(self) -> int:
        """Algorithmic bytes of msi_decode_attention per layer: K/V read + q read + o write."""
        return self.cache.kv_bytes_read() + 2 * self.T * self.n_heads * _lib.HEAD_DIM * 2


def request_cost_model(model, hbm_gbs: float = 6546.6, tflops: float = 1400.0):
    """perf_model.CostModel whose per-request attention cost is
    alpha * seq_len + beta: alpha = the KV bytes one cached token adds to the
    decode read (2 n_kv 128 x 2 B) at the HBM rate, beta = the request's
    projection FLOPs at the tensor rate."""
    from .perf_model import CostModel

    n_heads, n_kv = head_layout(model)
    alpha = 2 * n_kv * _lib.HEAD_DIM * 2 / (hbm_gbs * 1e9)
    beta = 2.0 * model.hidden * (n_heads + 2 * n_kv + n_heads) * _lib.HEAD_DIM / (tflops * 1e12)
    return CostModel(k1=alpha * 730 + beta, k2=0.0, k3=1e-6, k4=1e-4, alpha=alpha, beta=beta)


def composed_ctx_lens(model, n_a: int, b_a: int, avg_seq_len: int, seed: int = 0):
    """Attention batch composition over the data-parallel attention GPUs
    (balance.compose_attention_batches): a pool of n_a * b_a
    decode requests (uniform lengths, mean avg_seq_len, identical on every
    rank for a seed) is split into n_a batches of b_a requests whose predicted
    attention times are balanced (largest first onto the least-loaded GPU).  Returns (per-GPU ctx_lens, AttnBatchPlan)."""
    from .balance import compose_attention_batches

    lens = batch_composition(n_a * b_a, avg_seq_len, seed, "uniform")
    reqs = list(enumerate(lens.tolist()))
    plan = compose_attention_batches(reqs, n_a, request_cost_model(model), max_batch=b_a, mode="lpt")
    return plan.seq_lens(reqs), plan


class AttentionTPStage:
    """One micro-batch's attention stage on an attention node of tp_a GPUs
    (DeploymentPlan.tp_a > 1; csrc/attn_tp.cu).

    This GPU (rank r of its node) holds heads [r nh_l, (r+1) nh_l) and KV heads
    [r kv_l, (r+1) kv_l) of every node sequence (tp_a * T sequences: node
    token s*T + t is peer s's token t), and its own T-token shard of the
    residual stream -- its M2N batch.  forward(x_shard):

        msi_tp_publish   x -> symmetric shard buffer, release the node peers
        msi_tp_qkv       all-gather + QKV GEMM + RoPE/append in one kernel
        msi_decode_attention  this GPU's heads, all node tokens
        msi_tp_oproj     O projection, reduce-scatter in the epilogue
        msi_tp_reduce    y = bf16(x + sum of the tp_a partials)

    ``weights`` are the full AttentionWeights (identical on every node GPU);
    each GPU slices its heads.  ``ctx_lens`` are the node's tp_a * T cached
    lengths (identical on every node GPU, and so is the block table)."""

    def __init__(self, model, T: int, layers: int, group, slot: int, weights: AttentionWeights,
                 ctx_lens: np.ndarray, seed: int = 0, theta: float = ROPE_THETA, headroom: int = 0):
        g = group
        self.tp = g.plan.tp_a
        if self.tp < 2 or not g.is_attention:
            raise ValueError("AttentionTPStage needs an attention rank of a tp_a > 1 plan")
        if T > g.plan.b_a:
            raise ValueError("T exceeds the plan's b_a")
        self.g, self.model, self.T, self.slot, self.theta = g, model, T, slot, theta
        self.r = g.attn_index % self.tp
        n_heads, n_kv = weights.n_heads, weights.n_kv
        if n_kv % self.tp:
            raise ValueError(f"tp_a={self.tp} must divide the {n_kv} KV heads")
        self.n_heads, self.n_kv = n_heads // self.tp, n_kv // self.tp  # this GPU's heads
        D = _lib.HEAD_DIM
        r, hl, kl = self.r, self.n_heads, self.n_kv
        wq = weights.wqkv[:n_heads * D]
        wk = weights.wqkv[n_heads * D:(n_heads + n_kv) * D]
        wv = weights.wqkv[(n_heads + n_kv) * D:]
        self.wqkv = torch.cat([wq[r * hl * D:(r + 1) * hl * D], wk[r * kl * D:(r + 1) * kl * D],
                               wv[r * kl * D:(r + 1) * kl * D]]).contiguous()
        self.wo = weights.wo[:, r * hl * D:(r + 1) * hl * D].contiguous()
        ctx = np.asarray(ctx_lens, np.int32)
        if ctx.shape != (self.tp * T,):
            raise ValueError("ctx_lens must hold the node's tp_a * T sequences")
        # same seed on every node GPU -> same block table; KV contents per head slice
        self.cache = PagedKVCache(self.tp * T, kl, ctx, layers, g.device, seed, headroom=headroom)
        self.q = torch.empty((self.tp * T, hl, D), dtype=torch.bfloat16, device=g.device)
        self.o = torch.empty((self.tp * T, hl * D), dtype=torch.bfloat16, device=g.device)
        self.y = torch.empty((T, model.hidden), dtype=torch.bfloat16, device=g.device)
        self.ws = ops.decode_attention_workspace(self.tp * T, hl, kl, self.cache.max_pages, g.device)
        self.timing = None
        self.qkv_width = self.wqkv.shape[0]

    def forward(self, x: torch.Tensor, layer: int, out: torch.Tensor | None = None) -> torch.Tensor:
        """x bf16 [T, h] (this GPU's shard) -> x + Attn(x) W_o^T for the shard."""
        c, g, s = self.cache, self.g, ops._stream()
        out = self.y if out is None else out
        ctx = g.ctx
        _lib.call("msi_tp_publish", ctx, ops._ptr(x), self.T, self.slot, 0, s)
        _lib.call("msi_tp_qkv", ctx, ops._ptr(self.wqkv), self.n_heads, self.n_kv, ops._ptr(c.pos),
                  ctypes.c_float(self.theta), ops._ptr(c.block_table), c.block_table.shape[1], ops._ptr(c.k[layer]),
                  ops._ptr(c.v[layer]), ops._ptr(self.q), self.T, self.slot, 0, s)
        if self.timing is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True)
            e0.record()
        ops.decode_attention(self.q, c.k[layer], c.v[layer], c.block_table, c.lens, self.o, self.ws)
        if self.timing is not None:
            e1.record()
            self.timing.append((e0, e1))
        _lib.call("msi_tp_oproj", ctx, ops._ptr(self.o), ops._ptr(self.wo), self.o.shape[1], self.T, self.slot, 0, s)
        _lib.call("msi_tp_reduce", ctx, ops._ptr(x), ops._ptr(out), self.T, self.slot, 0, s)
        return out

    def flops(self) -> float:
        return 2.0 * self.tp * self.T * self.model.hidden * (self.qkv_width + self.o.shape[1])

    def attn_bytes(self) -> int:
        return self.cache.kv_bytes_read() + 2 * self.tp * self.T * self.n_heads * _lib.HEAD_DIM * 2
