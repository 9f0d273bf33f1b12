"""CPU oracle for the disaggregated-EP MoE decode step (numpy + liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py, as the checker.  The
product path never imports it.

PARITY UNPINNED BY THE REFERENCE.  The reference (/root/reference) ships no
implementation, tests or golden vectors for this path; this
oracle restates the paper's semantics with the build's precision contract:

* router   PAPER.md:83 (gate = x . W_g, top-K), PAPER.md:444-447 (fused top-K,
           per-expert counts, normalized weights, scatter) -> ``router``,
           ``place`` (bit-exact contract: idx, counts, slots, and weights via
           the deterministic exp in msi_oracle.c)
* dispatch PAPER.md:396-411 (M2N sender/receiver), per-pair bytes
           PAPER.md:632 -> ``dispatch_rows`` (bit-exact receive rows),
           ``dispatch_layout`` (the expert GEMM's virtual row order)
* expert   PAPER.md:285-286 (FFN in/out GEMMs) + SwiGLU per BASELINE
           north_star -> ``expert_ffn`` (fp32 accumulate; bf16 rounding at
           X, H, Y; tolerance-checked)
* expert TP (tp_e GPUs per expert node) ->
           ``expert_ffn_tp`` (per-rank h' slices, bf16 partials) and
           ``moe_layer(tp=)`` (the combine sums the partials, ascending (k, r))
* combine  PAPER.md:83, 97 -> ``combine`` (fp32 fmaf, ascending k; bit-exact
           given identical expert outputs)
* pipeline SPEC.md:237-272 -> paper_2504_02263_b200.pipeline (closed forms)

What *is* pinned by the reference -- the sizing numbers it states -- is
checked in tests/test_oracle.py (196,608 B per pair PAPER.md:632; gemm_flops
SPEC.md:127; P_e SPEC.md:153).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

ROW_ALIGN = 128  # per-expert segment alignment in the receive buffer (GEMM M tile)


def build() -> str:
    path = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "msi_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE], check=True, capture_output=True)
    return path


def lib():
    global _LIB
    if _LIB is None:
        L = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i = ctypes.c_int
        L.orc_router.argtypes = [P, P, i, i, i, i, P, P, P]
        L.orc_place.argtypes = [P, i, i, i, P, P]
        L.orc_combine.argtypes = [P, P, P, i, i, i, P]
        L.orc_combine.restype = None
        L.orc_bf16_round.argtypes = [P, P, ctypes.c_size_t]
        L.orc_bf16_round.restype = None
        L.orc_swiglu.argtypes = [P, P, P, ctypes.c_size_t]
        L.orc_swiglu.restype = None
        L.orc_decode_attention.argtypes = [P, P, P, P, i, P, i, i, i, ctypes.c_float, P]
        L.orc_decode_attention.restype = None
        L.orc_fill_normal.argtypes = [P, P, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_float]
        L.orc_fill_normal.restype = None
        L.msi_det_expf.argtypes = [ctypes.c_float]
        L.msi_det_expf.restype = ctypes.c_float
        _LIB = L
    return _LIB


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------- bf16 ---- #
def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns (uint16), round-to-nearest-even."""
    src = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(src.shape, dtype=np.uint16)
    lib().orc_bf16_round(_p(src), _p(out), src.size)
    return out


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def det_expf(d: float) -> float:
    return float(lib().msi_det_expf(float(d)))


# ------------------------------------------------------------- synthetic --- #
@dataclass
class LayerWeights:
    """Natural-layout bf16 weights (uint16 bit patterns)."""

    wg: np.ndarray      # [E, H]        gate (router) weights
    w_gate: np.ndarray  # [E, Hp, H]    FFN gate projection
    w_up: np.ndarray    # [E, Hp, H]    FFN up projection
    w_down: np.ndarray  # [E, H, Hp]    FFN down projection


def synth_weights(H: int, Hp: int, E: int, seed: int = 0, experts=None) -> LayerWeights:
    """SURVEY.md §8(d) init: W_g, W_gate, W_up ~ N(0, 1/H), W_down ~ N(0, 1/Hp),
    rounded to bf16.  ``experts`` limits the FFN weights to a subset (the CPU
    baseline samples)."""
    rng = np.random.default_rng(seed)
    wg = bf16_round(rng.standard_normal((E, H), dtype=np.float32) / np.sqrt(H))
    ids = range(E) if experts is None else experts
    n = len(list(ids))
    wgate = np.empty((n, Hp, H), np.uint16)
    wup = np.empty((n, Hp, H), np.uint16)
    wdown = np.empty((n, H, Hp), np.uint16)
    for j in range(n):
        wgate[j] = bf16_round(rng.standard_normal((Hp, H), dtype=np.float32) / np.sqrt(H))
        wup[j] = bf16_round(rng.standard_normal((Hp, H), dtype=np.float32) / np.sqrt(H))
        wdown[j] = bf16_round(rng.standard_normal((H, Hp), dtype=np.float32) / np.sqrt(Hp))
    return LayerWeights(wg, wgate, wup, wdown)


def synth_tokens(T: int, H: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return bf16_round(rng.standard_normal((T, H), dtype=np.float32))


# ---------------------------------------------------------------- router --- #
def router(x: np.ndarray, wg: np.ndarray, K: int, want_logits: bool = False):
    """x [T,H] bf16, wg [E,H] bf16 -> idx [T,K] int32, w [T,K] fp32 (and logits)."""
    x = np.ascontiguousarray(x, np.uint16)
    wg = np.ascontiguousarray(wg, np.uint16)
    T, H = x.shape
    E = wg.shape[0]
    idx = np.empty((T, K), np.int32)
    w = np.empty((T, K), np.float32)
    lg = np.empty((T, E), np.float32) if want_logits else None
    rc = lib().orc_router(_p(x), _p(wg), T, H, E, K, _p(idx), _p(w),
                          _p(lg) if lg is not None else None)
    if rc:
        raise ValueError(f"orc_router: bad shape (rc={rc}); H must be a multiple of 256")
    return (idx, w, lg) if want_logits else (idx, w)


def place(idx: np.ndarray, E: int):
    """-> cnt [E] int32, slot [T,K] int32 (ascending token order per expert)."""
    idx = np.ascontiguousarray(idx, np.int32)
    T, K = idx.shape
    cnt = np.empty(E, np.int32)
    slot = np.empty((T, K), np.int32)
    if lib().orc_place(_p(idx), T, K, E, _p(cnt), _p(slot)):
        raise ValueError("orc_place: expert index out of range")
    return cnt, slot


def physical_slots(idx: np.ndarray, rep: np.ndarray, sender: int) -> np.ndarray:
    """Replicated experts: token t of sender s routed to
    logical expert e goes to replica (t + s) mod rep[e, 0], i.e. physical slot
    rep[e, 1 + r] -- the rule msi_gate_topk_placed implements."""
    idx = np.asarray(idx, np.int64)
    t = np.arange(idx.shape[0])[:, None]
    r = (t + sender) % rep[idx, 0]
    return rep[idx, 1 + r].astype(np.int32)


# -------------------------------------------------------------- dispatch --- #
def segment_starts(total: np.ndarray, align: int = ROW_ALIGN) -> np.ndarray:
    """Start row of each local expert's segment: segments are packed in expert
    order, each start aligned to ``align`` rows (the GEMM M tile)."""
    padded = (np.asarray(total, np.int64) + align - 1) // align * align
    return np.concatenate([[0], np.cumsum(padded)[:-1]]).astype(np.int64)


def dispatch_layout(cnt_all: np.ndarray, E_l: int):
    """cnt_all [n_a, E] -> per expert GPU q: (total [E_l], seg_start [E_l],
    base [n_a, E_l]): the expert GEMM's *virtual* rows -- expert e_l's rows
    are its senders' rows in ascending (sender, slot) order, segments 128-row
    aligned (the activation buffer hbuf uses this order)."""
    cnt_all = np.asarray(cnt_all, np.int64)
    n_a, E = cnt_all.shape
    out = []
    for q in range(E // E_l):
        c = cnt_all[:, q * E_l:(q + 1) * E_l]
        total = c.sum(0)
        base = np.cumsum(c, 0) - c
        out.append((total, segment_starts(total), base))
    return out


def dispatch_rows(idx: np.ndarray, slot: np.ndarray, s: int, E_l: int, n_a: int, cap_s: int):
    """Destination (expert GPU, receive row) of every (t, k) of sender s
    (PAPER.md:396-411): the receive buffer of an expert GPU has one region of
    cap_s (= b_a) rows per (local expert e_l, sender), at row
    (e_l * n_a + s) * cap_s; row (t, k) sits at its slot inside it.  A sender
    therefore places its rows from its own counts alone."""
    idx = np.asarray(idx, np.int64)
    q = idx // E_l
    rows = ((idx % E_l) * n_a + s) * cap_s + np.asarray(slot, np.int64)
    return q.astype(np.int32), rows


# ---------------------------------------------------------------- expert --- #
def expert_ffn(xe: np.ndarray, w_gate: np.ndarray, w_up: np.ndarray,
               w_down: np.ndarray) -> np.ndarray:
    """One expert's SwiGLU FFN on its rows.  xe [t,H] bf16 -> y [t,H] bf16.
    G, U fp32-accumulated; H = bf16(silu(G) * U); Y = bf16(H . W_down^T)."""
    if xe.shape[0] == 0:
        return np.zeros((0, w_down.shape[0]), np.uint16)
    xf = bf16_to_f32(xe)
    g = xf @ bf16_to_f32(w_gate).T
    u = xf @ bf16_to_f32(w_up).T
    h = np.empty(g.shape, np.uint16)
    g = np.ascontiguousarray(g, np.float32)
    u = np.ascontiguousarray(u, np.float32)
    lib().orc_swiglu(_p(g), _p(u), _p(h), g.size)
    y = bf16_to_f32(h) @ bf16_to_f32(w_down).T
    return bf16_round(y)


def expert_ffn_tp(xe: np.ndarray, w_gate: np.ndarray, w_up: np.ndarray, w_down: np.ndarray,
                  tp: int) -> np.ndarray:
    """Expert tensor parallelism over h' (config.DeploymentPlan.tp_e): TP rank
    r owns features [r h'/tp, (r+1) h'/tp) and returns the bf16 partial
    y_r = bf16(H_r . W_down[:, F_r]^T).  xe [t,H] -> [t, tp, H]."""
    Hp = w_gate.shape[0]
    f = Hp // tp
    parts = [expert_ffn(xe, w_gate[r * f:(r + 1) * f], w_up[r * f:(r + 1) * f], w_down[:, r * f:(r + 1) * f])
             for r in range(tp)]
    return np.stack(parts, axis=1)


# --------------------------------------------------------------- combine --- #
def combine(y: np.ndarray, w: np.ndarray, resid: np.ndarray | None = None) -> np.ndarray:
    """y [T,K,H] bf16, w [T,K] fp32 -> out [T,H] bf16 (optional residual)."""
    y = np.ascontiguousarray(y, np.uint16)
    w = np.ascontiguousarray(w, np.float32)
    T, K, H = y.shape
    out = np.empty((T, H), np.uint16)
    r = None if resid is None else np.ascontiguousarray(resid, np.uint16)
    lib().orc_combine(_p(y), _p(w), _p(r) if r is not None else None, T, K, H, _p(out))
    return out


# ------------------------------------------------------------ full layer --- #
@dataclass
class LayerResult:
    idx: list      # per sender [T,K]
    w: list        # per sender [T,K]
    cnt: np.ndarray  # [n_a, E]
    slot: list     # per sender [T,K]
    layout: list   # per expert GPU (total, seg_start, base)
    y: list        # per sender [T,K,H] expert outputs (unweighted)
    out: list      # per sender [T,H]


def moe_layer(xs: list, wts: LayerWeights, K: int, n_e: int, resid: bool = False,
              rep: np.ndarray | None = None, phys2log: np.ndarray | None = None, tp: int = 1) -> LayerResult:
    """Full MoE layer step for n_a senders (one micro-batch): route, place,
    dispatch, SwiGLU experts, combine.  With a replica table ``rep`` [E, R+1]
    and ``phys2log`` [P] the placement, counts and receive layout are per
    physical slot (``idx`` stays logical; ``LayerResult.pidx`` holds the
    slots); every slot runs its logical expert's weights.  ``tp`` > 1: expert
    tensor parallelism -- n_e expert GPUs form n_e / tp nodes (the layout is
    per node), ``y`` holds the tp partials [T, K, tp, H] and the combine sums
    them in ascending (k, r) order."""
    E = wts.wg.shape[0]
    P = E if rep is None else len(phys2log)
    E_l = P // (n_e // tp)
    H = wts.wg.shape[1]
    idxs, ws, slots, cnts, pidxs = [], [], [], [], []
    for s_, x in enumerate(xs):
        i, w = router(x, wts.wg, K)
        pi = i if rep is None else physical_slots(i, rep, s_)
        c, s = place(pi, P)
        idxs.append(i), ws.append(w), slots.append(s), cnts.append(c), pidxs.append(pi)
    cnt = np.stack(cnts)
    layout = dispatch_layout(cnt, E_l)
    # gather each slot's rows in receive order, run its expert, scatter back
    ys = [np.empty((x.shape[0], K, tp, H), np.uint16) for x in xs]
    for p in range(P):
        e = p if rep is None else int(phys2log[p])
        srcs = []
        for s_, (pi, sl) in enumerate(zip(pidxs, slots)):
            t, k = np.nonzero(pi == p)
            order = np.argsort(sl[t, k], kind="stable")
            srcs.append((s_, t[order], k[order]))
        if e < 0 or not any(len(t) for _, t, _ in srcs):
            continue
        rows = np.concatenate([xs[s_][t] for s_, t, _ in srcs])
        y = expert_ffn_tp(rows, wts.w_gate[e], wts.w_up[e], wts.w_down[e], tp)
        off = 0
        for s_, t, k in srcs:
            ys[s_][t, k] = y[off:off + len(t)]
            off += len(t)
    outs = [combine(y.reshape(y.shape[0], K * tp, H), np.repeat(w, tp, axis=1), x if resid else None)
            for y, w, x in zip(ys, ws, xs)]
    if tp == 1:
        ys = [y[:, :, 0] for y in ys]
    res = LayerResult(idxs, ws, cnt, slots, layout, ys, outs)
    res.pidx = pidxs
    return res


# -------------------------------------------------------- sizing (pins) ---- #
def pair_payload_bytes(b: int, K: int, E: int, h: int, tp_a: int = 1, bytes_per=2) -> float:
    """Average sender->receiver bytes (PAPER.md:632 example)."""
    return b * K / E * h * bytes_per / tp_a


def gemm_flops(b: int, h_in: int, h_out: int) -> int:
    """2 * b * h_in * h_out."""
    if min(b, h_in, h_out) <= 0:
        raise ValueError("gemm_flops: all dimensions must be > 0")
    return 2 * b * h_in * h_out


def expert_param_bytes(layers: int, h: int, hp: int, bytes_per: int = 2, swiglu: bool = False) -> int:
    """P_e: L * 2 * h * h' * bytes (3 matrices with SwiGLU)."""
    return layers * (3 if swiglu else 2) * h * hp * bytes_per


# ------------------------------------------------------- attention stage --- #
# SURVEY.md §8(f) rank 3.  The reference only models this stage (T_a = k1 b_a
# + k2, KV traffic 2 b s h bytes / g: SPEC.md:156-164, 186; Table 3 GEMMs
# PAPER.md:283-284); the restatement below is the standard GQA decode layer
# those formulas describe: QKV projection (h -> h (1 + 2/g)), RoPE, KV append,
# softmax(q K^T / sqrt(d)) V over the cached tokens, output projection
# (h -> h) plus residual.  fp32 math, bf16 rounding where the GPU path stores
# (qkv, rotated q/k, attention output, stage output).
KV_PAGE = 64
HEAD_DIM = 128


def rope(x: np.ndarray, pos: np.ndarray, theta: float) -> np.ndarray:
    """Rotate-half RoPE.  x fp32 [T, heads, 128], pos int [T] -> fp32."""
    d = x.shape[-1]
    i = np.arange(d // 2, dtype=np.float32)
    inv = (np.float32(1.0) / np.power(np.float32(theta), (2 * i) / np.float32(d))).astype(np.float32)
    ang = (pos.astype(np.float32)[:, None] * inv[None, :]).astype(np.float32)
    cs, sn = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    lo, hi = x[..., : d // 2], x[..., d // 2:]
    return np.concatenate([lo * cs - hi * sn, hi * cs + lo * sn], axis=-1).astype(np.float32)


def paged_kv_gather(cache: np.ndarray, block_table: np.ndarray, t: int, n: int, kvh: int) -> np.ndarray:
    """Rows 0..n-1 of sequence t's KV head kvh from a paged cache
    [pages, n_kv, 64, 128] (bf16 bits) -> fp32 [n, 128]."""
    pages = (n + KV_PAGE - 1) // KV_PAGE
    rows = np.concatenate([cache[block_table[t, p], kvh] for p in range(pages)]) if pages else \
        np.zeros((0, HEAD_DIM), np.uint16)
    return bf16_to_f32(rows[:n])


def decode_attention(q: np.ndarray, k_cache: np.ndarray, v_cache: np.ndarray, block_table: np.ndarray,
                     seq_lens: np.ndarray, scale: float | None = None) -> np.ndarray:
    """q bf16 [T, n_heads, 128]; caches bf16 [pages, n_kv, 64, 128] -> out bf16
    [T, n_heads * 128].  An empty sequence yields zeros."""
    T, nh, d = q.shape
    n_kv = k_cache.shape[1]
    G = nh // n_kv
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    qf = bf16_to_f32(q)
    out = np.zeros((T, nh, d), np.float32)
    for t in range(T):
        n = int(seq_lens[t])
        if n == 0:
            continue
        for h in range(n_kv):
            K = paged_kv_gather(k_cache, block_table, t, n, h)
            V = paged_kv_gather(v_cache, block_table, t, n, h)
            s = (qf[t, h * G:(h + 1) * G] @ K.T) * np.float32(scale)
            s = s - s.max(axis=1, keepdims=True)
            p = np.exp(s)
            out[t, h * G:(h + 1) * G] = (p @ V) / p.sum(axis=1, keepdims=True)
    return bf16_round(out.reshape(T, nh * d))


def rope_append(qkv: np.ndarray, pos: np.ndarray, n_heads: int, n_kv: int, theta: float,
                block_table: np.ndarray, k_cache: np.ndarray, v_cache: np.ndarray) -> np.ndarray:
    """qkv bf16 [T, (n_heads + 2 n_kv) 128]; rotates q, k at pos and writes k, v
    into the caches in place.  Returns rotated q bf16 [T, n_heads, 128]."""
    T = qkv.shape[0]
    f = bf16_to_f32(qkv)
    q = rope(f[:, : n_heads * HEAD_DIM].reshape(T, n_heads, HEAD_DIM), pos, theta)
    k = rope(f[:, n_heads * HEAD_DIM:(n_heads + n_kv) * HEAD_DIM].reshape(T, n_kv, HEAD_DIM), pos, theta)
    v = qkv[:, (n_heads + n_kv) * HEAD_DIM:(n_heads + 2 * n_kv) * HEAD_DIM].reshape(T, n_kv, HEAD_DIM)
    kb = bf16_round(k)
    for t in range(T):
        pg, r = block_table[t, pos[t] // KV_PAGE], pos[t] % KV_PAGE
        k_cache[pg, :, r] = kb[t]
        v_cache[pg, :, r] = v[t]
    return bf16_round(q)


def attention_stage(x: np.ndarray, wqkv: np.ndarray, wo: np.ndarray, pos: np.ndarray, n_heads: int, n_kv: int,
                    theta: float, block_table: np.ndarray, k_cache: np.ndarray, v_cache: np.ndarray) -> np.ndarray:
    """One decode attention layer on the attention GPU: x bf16 [T, h] ->
    bf16(x + attn(x) W_o^T).  Appends the new token at pos (caches updated in place)."""
    qkv = bf16_round(bf16_to_f32(x) @ bf16_to_f32(wqkv).T)
    q = rope_append(qkv, pos, n_heads, n_kv, theta, block_table, k_cache, v_cache)
    o = decode_attention(q, k_cache, v_cache, block_table, pos.astype(np.int64) + 1)
    return bf16_round(bf16_to_f32(x) + bf16_to_f32(o) @ bf16_to_f32(wo).T)


def decode_attention_c(q: np.ndarray, k_cache: np.ndarray, v_cache: np.ndarray, block_table: np.ndarray,
                       seq_lens: np.ndarray, scale: float | None = None) -> np.ndarray:
    """``decode_attention`` in C (OpenMP over (sequence, KV head)): same fp32
    math, different summation order (tests/test_oracle.py checks agreement).
    Used by the CPU baseline, which runs the whole attention stage."""
    q = np.ascontiguousarray(q, np.uint16)
    T, nh, d = q.shape
    if d != HEAD_DIM:
        raise ValueError("head dim must be 128")
    n_kv = k_cache.shape[1]
    if nh % n_kv or nh // n_kv > 16:
        raise ValueError("need n_heads = G * n_kv with G <= 16")
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    bt = np.ascontiguousarray(block_table, np.int32)
    lens = np.ascontiguousarray(seq_lens, np.int32)
    out = np.empty((T, nh * d), np.uint16)
    lib().orc_decode_attention(_p(q), _p(np.ascontiguousarray(k_cache)), _p(np.ascontiguousarray(v_cache)),
                               _p(bt), bt.shape[1], _p(lens), T, nh, n_kv, float(scale), _p(out))
    return out


def fill_normal(shape, seed: int, scale: float = 1.0, as_f32: bool = False) -> np.ndarray:
    """N(0, scale^2) rounded to bf16 (uint16 bits, or the same values as fp32),
    generated in parallel in C (synthetic inputs for the CPU baseline)."""
    n = int(np.prod(shape))
    if as_f32:
        out = np.empty(shape, np.float32)
        lib().orc_fill_normal(_p(out), None, n, seed, float(scale))
    else:
        out = np.empty(shape, np.uint16)
        lib().orc_fill_normal(None, _p(out), n, seed, float(scale))
    return out


# ------------------------------------------------- CPU baseline layer ------ #
class CpuDecodeLayer:
    """The bench's decode layer step on the host cores (the CPU baseline the
    GPU path is timed against; the reference ships no implementation of the
    path): for T tokens of one attention GPU's step, the whole
    co-located layer with the oracle's arithmetic --

      attention stage  x W_qkv^T, RoPE + paged-KV append, GQA decode over the
                       paged cache (``decode_attention_c``), + x + o W_o^T
      router           ``router`` + ``place`` (bit-exact contract)
      experts          SwiGLU of every expert over its routed rows (fp32 BLAS,
                       bf16 rounding at H and Y)
      combine          ``combine`` with the attention output as residual

    Weights are held as fp32 copies of bf16 values (a CPU keeps its GEMM
    operands in the format its BLAS runs); the KV cache is bf16 pages.  No
    part of a step is sampled or projected."""

    def __init__(self, H: int, Hp: int, E: int, K: int, T: int, n_heads: int, n_kv: int,
                 ctx: np.ndarray, theta: float = 1e6, seed: int = 0):
        self.H, self.Hp, self.E, self.K, self.T = H, Hp, E, K, T
        self.n_heads, self.n_kv, self.theta = n_heads, n_kv, theta
        s = seed * 1000
        self.wg = fill_normal((E, H), s + 1, 1.0 / np.sqrt(H))
        self.w_gate = [fill_normal((Hp, H), s + 10 + e, 1.0 / np.sqrt(H), as_f32=True) for e in range(E)]
        self.w_up = [fill_normal((Hp, H), s + 100 + e, 1.0 / np.sqrt(H), as_f32=True) for e in range(E)]
        self.w_down = [fill_normal((H, Hp), s + 200 + e, 1.0 / np.sqrt(Hp), as_f32=True) for e in range(E)]
        width = (n_heads + 2 * n_kv) * HEAD_DIM
        self.wqkv = fill_normal((width, H), s + 300, 1.0 / np.sqrt(H), as_f32=True)
        self.wo = fill_normal((H, n_heads * HEAD_DIM), s + 301, 1.0 / np.sqrt(n_heads * HEAD_DIM), as_f32=True)
        self.ctx = np.asarray(ctx, np.int32)
        need = (self.ctx.astype(np.int64) + 1 + KV_PAGE - 1) // KV_PAGE
        self.pages = int(need.sum())
        rng = np.random.default_rng(seed + 7919)
        perm = rng.permutation(self.pages).astype(np.int32)
        self.bt = np.zeros((T, int(need.max())), np.int32)
        off = 0
        for t in range(T):
            self.bt[t, : need[t]] = perm[off: off + need[t]]
            off += need[t]
        self.k_cache = fill_normal((self.pages, n_kv, KV_PAGE, HEAD_DIM), s + 400)
        self.v_cache = fill_normal((self.pages, n_kv, KV_PAGE, HEAD_DIM), s + 401)

    def attention(self, x: np.ndarray) -> np.ndarray:
        qkv = bf16_round(bf16_to_f32(x) @ self.wqkv.T)
        q = rope_append(qkv, self.ctx, self.n_heads, self.n_kv, self.theta, self.bt, self.k_cache, self.v_cache)
        o = decode_attention_c(q, self.k_cache, self.v_cache, self.bt, self.ctx.astype(np.int64) + 1)
        return bf16_round(bf16_to_f32(x) + bf16_to_f32(o) @ self.wo.T)

    def moe(self, h: np.ndarray) -> np.ndarray:
        idx, w = router(h, self.wg, self.K)
        cnt, slot = place(idx, self.E)
        y = np.zeros((h.shape[0], self.K, self.H), np.uint16)
        hf = bf16_to_f32(h)
        for e in range(self.E):
            t, k = np.nonzero(idx == e)
            if len(t) == 0:
                continue
            order = np.argsort(slot[t, k], kind="stable")  # receive order
            t, k = t[order], k[order]
            xe = hf[t]
            g = np.ascontiguousarray(xe @ self.w_gate[e].T)
            u = np.ascontiguousarray(xe @ self.w_up[e].T)
            act = np.empty(g.shape, np.uint16)
            lib().orc_swiglu(_p(g), _p(u), _p(act), g.size)
            y[t, k] = bf16_round(bf16_to_f32(act) @ self.w_down[e].T)
        return combine(y, w, h)

    def step(self, x: np.ndarray) -> tuple[np.ndarray, dict]:
        """One layer step: x bf16 [T, H] -> layer output bf16 [T, H] and the
        per-phase seconds."""
        import time
        t0 = time.perf_counter()
        h = self.attention(x)
        t1 = time.perf_counter()
        out = self.moe(h)
        t2 = time.perf_counter()
        return out, {"attention_s": t1 - t0, "moe_s": t2 - t1, "layer_s": t2 - t0}
