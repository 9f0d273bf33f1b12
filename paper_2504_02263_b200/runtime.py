"""Host runtime: roles, M2N group setup and the ping-pong decode step.

Python API of the path, one process per GPU:

* ``M2NGroup(model, plan, rank)`` -- creates this rank's libmsinfer context,
  exchanges CUDA IPC handles of the symmetric heaps with every peer (the
  paper's "pre-registered tensor") and maps them;
* ``MoEDecodeLayer`` -- ``router(x)``, ``dispatch(x, route, mb)``,
  ``expert_step(mb)``, ``combine(handle, resid)``: the four operations of one
  MoE layer;
* ``PingPongRunner`` -- the m-micro-batch x L-layer schedule of PAPER.md:219-238
  (Figure 4) expressed as per-rank program order on one CUDA stream; ordering
  across GPUs is carried only by device-side epoch counters, so the host never
  waits inside an iteration.  Phase timings use the SPEC timeline schema
  (attn, disp, ffn, comb).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

from . import _lib, ops
from .config import DeploymentPlan, MoeModelSpec, as_model_spec


# ----------------------------------------------------------------- helpers --
class _DevArray:
    """Zero-copy torch view of a device pointer owned by libmsinfer."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def device_view(ptr: int, shape, dtype: torch.dtype, device) -> torch.Tensor:
    typestr = {torch.bfloat16: "<u2", torch.int32: "<i4", torch.int64: "<i8",
               torch.uint8: "|u1"}[dtype]
    t = torch.as_tensor(_DevArray(ptr, shape, typestr), device=device)
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t


def make_plan_struct(model: MoeModelSpec, plan: DeploymentPlan, slots=None) -> _lib.Plan:
    """C plan for this deployment.  With a ``balance.SlotPlacement`` the M2N
    layer works on its P physical expert slots instead of the E logical experts."""
    if slots is None:
        plan.check_model(model)
    elif slots.E != model.experts or slots.n_e != plan.n_e:
        raise ValueError("slot placement does not match the model / plan")
    if plan.world > _lib.MAX_RANKS:
        raise ValueError(f"plan needs {plan.world} ranks; at most {_lib.MAX_RANKS} per box")
    p = _lib.Plan()
    p.world = plan.world
    p.n_a, p.n_e = plan.n_a, plan.n_e
    for i, r in enumerate(plan.attention_ranks()):
        p.attn_ranks[i] = r
    for i, r in enumerate(plan.expert_ranks()):
        p.expert_ranks[i] = r
    p.hidden, p.inter = model.hidden, model.intermediate
    p.experts, p.topk = (model.experts if slots is None else slots.P), model.topk
    p.max_tokens, p.slots = plan.b_a, plan.m
    p.tp_e = plan.tp_e
    p.tp_a = plan.tp_a
    return p


def exchange_blobs(blob: bytes, group=None) -> list[bytes]:
    """All-gather one bytes object per rank (torch.distributed; works on gloo
    and nccl).  Single-process use returns [blob]."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return [blob]
    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out


# ------------------------------------------------------------------ group ---
class M2NGroup:
    """This rank's M2N endpoint: context, peer mapping, role."""

    def __init__(self, model, plan: DeploymentPlan, rank: int = 0, device=None, group=None,
                 timeout_s: float = 20.0, slots=None):
        self.model = as_model_spec(model)
        self.plan = plan
        self.rank = rank
        self.role = plan.role_of(rank)
        self.slots = slots  # balance.SlotPlacement (replicated experts) or None
        self.device = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
        lib = _lib.load()
        _lib.call("msi_check_device")
        self._pstruct = make_plan_struct(self.model, plan, slots)
        ctx = ctypes.c_void_p()
        _lib.call("msi_ctx_create", ctypes.byref(self._pstruct), rank, ctypes.byref(ctx))
        self.ctx = ctx
        _lib.call("msi_set_wait_timeout", ctx, int(timeout_s * 1e9))
        h = _lib.IpcHandle()
        _lib.call("msi_ctx_export", ctx, ctypes.byref(h))
        blobs = exchange_blobs(bytes(h.bytes), group)
        if len(blobs) != plan.world:
            raise RuntimeError(f"process group has {len(blobs)} ranks, plan needs {plan.world}")
        for r, b in enumerate(blobs):
            if r == rank:
                continue
            hh = _lib.IpcHandle()
            ctypes.memmove(hh.bytes, b, _lib.IPC_HANDLE_BYTES)
            _lib.call("msi_ctx_import", ctx, r, ctypes.byref(hh))
        _lib.call("msi_ctx_finalize", ctx)
        exchange_blobs(b"ready", group)  # barrier: every heap zeroed before first use
        self.lib = lib
        self.is_attention = self.role in ("attention", "both")
        self.is_expert = self.role in ("expert", "both")
        self.attn_index = plan.attention_ranks().index(rank) if self.is_attention else -1
        self.expert_index = plan.expert_ranks().index(rank) if self.is_expert else -1
        if slots is not None and plan.tp_e != 1:
            raise ValueError("replicated placements with expert TP are not supported")
        self.E_l = plan.experts_per_gpu(self.model) if slots is None else slots.P_l  # local (physical) slots
        self.tp = plan.tp_e  # expert TP: this GPU holds h'/tp of each local expert
        self.tp_rank = self.expert_index % plan.tp_e if self.is_expert else 0
        self.node = self.expert_index // plan.tp_e if self.is_expert else -1
        self.P = self.model.experts if slots is None else slots.P
        ws = ctypes.c_void_p()
        nb = ctypes.c_size_t()
        _lib.call("msi_ctx_workspace", ctx, ctypes.byref(ws), ctypes.byref(nb))
        self.workspace_ptr = ws.value

    def buffer(self, which: int, slot: int) -> tuple[int, int]:
        p = ctypes.c_void_p()
        n = ctypes.c_size_t()
        _lib.call("msi_ctx_buffer", self.ctx, which, slot, ctypes.byref(p), ctypes.byref(n))
        return p.value, n.value

    def recv_view(self, slot: int) -> torch.Tensor:
        ptr, n = self.buffer(_lib.BUF_RECV, slot)
        H = self.model.hidden
        return device_view(ptr, (n // (2 * H), H), torch.bfloat16, self.device)

    def cntab_view(self, slot: int) -> torch.Tensor:
        ptr, n = self.buffer(_lib.BUF_CNTAB, slot)
        return device_view(ptr, (self.plan.n_a, self.model.experts), torch.int64, self.device)

    def status(self) -> int:
        s = ctypes.c_int32()
        _lib.call("msi_poll_status", self.ctx, ctypes.byref(s))
        return s.value

    def stats(self) -> tuple[int, int]:
        """(rows through expert FFN, FFN calls) since finalize (expert role)."""
        r, c = ctypes.c_uint64(), ctypes.c_uint64()
        _lib.call("msi_ctx_stats", self.ctx, ctypes.byref(r), ctypes.byref(c))
        return r.value, c.value

    TRACE_SLOTS = {0: "disp_start", 1: "disp_counts", 2: "disp_release", 3: "echo_start",
                   4: "echo_rows", 5: "echo_release", 6: "comb_start", 7: "comb_rows", 8: "comb_end",
                   9: "ffn_start", 10: "ffn_rows", 13: "gemm2_start", 14: "ffn_release"}

    def set_trace(self, on: bool = True):
        _lib.call("msi_set_trace", self.ctx, int(on))

    def trace(self) -> dict:
        """%globaltimer stamps (ns) of this rank's last traced phases."""
        buf = (ctypes.c_uint64 * 32)()
        _lib.call("msi_ctx_trace", self.ctx, buf, 32)
        return {name: buf[i] for i, name in self.TRACE_SLOTS.items() if buf[i]}

    def close(self):
        if getattr(self, "ctx", None):
            _lib.load().msi_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------- layer ----
@dataclass
class Route:
    """Router output for one micro-batch on an attention GPU."""

    idx: torch.Tensor   # [T,K] logical experts
    w: torch.Tensor     # [T,K] combine weights
    cnt: torch.Tensor   # [P] tokens per physical expert slot (= logical without replication)
    slot: torch.Tensor  # [T,K] rank within the physical slot
    T: int
    mb: int = 0
    epoch: int = 0
    pidx: torch.Tensor | None = None  # [T,K] physical slots (replicated experts) or None

    @property
    def dest(self) -> torch.Tensor:
        """Physical slot of every (t, k): what the M2N dispatch routes by."""
        return self.idx if self.pidx is None else self.pidx


class MoEDecodeLayer:
    """One MoE layer of the disaggregated decode step on this rank.

    Attention ranks hold ``wg`` [E, H]; expert ranks hold their local experts'
    ``w13`` [E_l, 2H', H] (ops.pack_w13 layout) and ``w2`` [E_l, H, H'].
    """

    def __init__(self, group: M2NGroup, wg: torch.Tensor | None = None,
                 w13: torch.Tensor | None = None, w2: torch.Tensor | None = None):
        self.g = group
        m = group.model
        if group.is_attention:
            if wg is None or tuple(wg.shape) != (m.experts, m.hidden):
                raise ValueError("attention ranks need wg [E, H]")
        if group.is_expert and (w13 is not None or w2 is not None):
            # (weights may be omitted on an expert rank that only runs expert_echo)
            E_l, hs = group.E_l, m.intermediate // group.tp  # expert TP: this GPU's h' slice
            if w13 is None or tuple(w13.shape) != (E_l, 2 * hs, m.hidden):
                raise ValueError(f"expert ranks need w13 [{E_l}, {2 * hs}, {m.hidden}]")
            if w2 is None or tuple(w2.shape) != (E_l, m.hidden, hs):
                raise ValueError(f"expert ranks need w2 [{E_l}, {m.hidden}, {hs}]")
        self.wg, self.w13, self.w2 = wg, w13, w2
        # epochs: 0 = "next use of the slot" counted on the device (default;
        # required inside CUDA graphs, whose replays the host cannot count).
        # device_epochs=False passes the host count explicitly; the kernels
        # check it against the device count and fail (status MSI_ESTATE) on a
        # mismatch instead of racing.
        self.device_epochs = True
        self.epoch_a = [0] * group.plan.m   # uses of each slot (attention side)
        self.epoch_e = [0] * group.plan.m   # uses of each slot (expert side)
        self._routes = []
        self._rep = None
        if group.is_attention:
            dev, K, T = group.device, m.topk, group.plan.b_a
            sl = group.slots
            if sl is not None:
                self._rep = torch.from_numpy(sl.rep.astype("int32").ravel()).to(dev)
            for _ in range(group.plan.m):
                self._routes.append(Route(torch.empty((T, K), dtype=torch.int32, device=dev),
                                          torch.empty((T, K), dtype=torch.float32, device=dev),
                                          torch.empty((group.P,), dtype=torch.int32, device=dev),
                                          torch.empty((T, K), dtype=torch.int32, device=dev), T,
                                          pidx=None if sl is None else
                                          torch.empty((T, K), dtype=torch.int32, device=dev)))
        self._ws = group.workspace_ptr

    # -- (1) router ---------------------------------------------------------
    def router(self, x: torch.Tensor, mb: int = 0, stream=None) -> Route:
        m = self.g.model
        T = x.shape[0]
        if T > self.g.plan.b_a:
            raise ValueError(f"micro-batch of {T} tokens exceeds plan.b_a={self.g.plan.b_a}")
        r = self._routes[mb]
        if self._rep is None:
            _lib.call("msi_gate_topk", ops._ptr(x), ops._ptr(self.wg), T, m.hidden, m.experts, m.topk,
                      ops._ptr(r.idx), ops._ptr(r.w), ops._ptr(r.cnt), ops._ptr(r.slot),
                      ctypes.c_void_p(self._ws), ops._stream(stream))
        else:  # replicated experts: route to physical slots (balance.SlotPlacement)
            sl = self.g.slots
            _lib.call("msi_gate_topk_placed", ops._ptr(x), ops._ptr(self.wg), T, m.hidden, m.experts, m.topk,
                      ops._ptr(self._rep), sl.R, sl.P, self.g.attn_index, ops._ptr(r.idx), ops._ptr(r.pidx),
                      ops._ptr(r.w), ops._ptr(r.cnt), ops._ptr(r.slot), ctypes.c_void_p(self._ws),
                      ops._stream(stream))
        r.T, r.mb = T, mb
        return r

    # -- (1) fused router + M2N dispatch ---------------------
    def route_dispatch(self, x: torch.Tensor, mb: int = 0, stream=None) -> Route:
        """router(x) and dispatch in one launch (msi_route_dispatch): every
        routed row is stored into its expert GPU's receive region by the CTA
        that routed it.  Same outputs as router() + dispatch()."""
        m = self.g.model
        T = x.shape[0]
        if T > self.g.plan.b_a:
            raise ValueError(f"micro-batch of {T} tokens exceeds plan.b_a={self.g.plan.b_a}")
        r = self._routes[mb]
        self.epoch_a[mb] += 1
        r.T, r.mb, r.epoch = T, mb, (0 if self.device_epochs else self.epoch_a[mb])
        if self._rep is None:
            _lib.call("msi_route_dispatch", self.g.ctx, ops._ptr(x), ops._ptr(self.wg), T, m.experts, None, 0,
                      ops._ptr(r.idx), None, ops._ptr(r.w), ops._ptr(r.cnt), ops._ptr(r.slot), mb, r.epoch,
                      ops._stream(stream))
        else:
            _lib.call("msi_route_dispatch", self.g.ctx, ops._ptr(x), ops._ptr(self.wg), T, m.experts,
                      ops._ptr(self._rep), self.g.slots.R, ops._ptr(r.idx), ops._ptr(r.pidx), ops._ptr(r.w),
                      ops._ptr(r.cnt), ops._ptr(r.slot), mb, r.epoch, ops._stream(stream))
        return r

    # -- (1) M2N dispatch -----------------------------------------------------
    def dispatch(self, x: torch.Tensor, route: Route, mb: int | None = None, stream=None) -> Route:
        mb = route.mb if mb is None else mb
        self.epoch_a[mb] += 1
        route.mb, route.epoch = mb, (0 if self.device_epochs else self.epoch_a[mb])
        _lib.call("msi_dispatch", self.g.ctx, ops._ptr(x), ops._ptr(route.cnt), ops._ptr(route.dest),
                  ops._ptr(route.slot), route.T, mb, route.epoch, ops._stream(stream))
        return route

    # -- (2) expert FFN -------------------------------------------------------
    def expert_step(self, mb: int = 0, stream=None) -> int:
        """Wait for the slot's rows (msi_expert_wait), then the SwiGLU FFN
        (msi_expert_ffn: GEMM1 + GEMM2 whose epilogue is the N2M send)."""
        self.expert_wait(mb, stream)
        return self.expert_ffn(mb, stream)

    def expert_wait(self, mb: int = 0, stream=None):
        if os.environ.get("MSI_EXPERT_WAIT", "1") == "0":  # A/B switch: rely on GEMM1's own wait
            return
        epoch = 0 if self.device_epochs else self.epoch_e[mb] + 1
        _lib.call("msi_expert_wait", self.g.ctx, mb, epoch, ops._stream(stream))

    def expert_ffn(self, mb: int = 0, stream=None) -> int:
        if self.w13 is None or self.w2 is None:
            raise ValueError("expert_step needs w13/w2 on this expert rank")
        self.epoch_e[mb] += 1
        _lib.call("msi_expert_ffn", self.g.ctx, ops._ptr(self.w13), ops._ptr(self.w2), mb,
                  0 if self.device_epochs else self.epoch_e[mb], ops._stream(stream))
        return self.epoch_e[mb]

    def expert_echo(self, mb: int = 0, stream=None) -> int:
        """Identity expert: the N2M leg without the FFN (M2N measurements)."""
        self.epoch_e[mb] += 1
        _lib.call("msi_expert_echo", self.g.ctx, mb, 0 if self.device_epochs else self.epoch_e[mb],
                  ops._stream(stream))
        return self.epoch_e[mb]

    # -- (3) N2M combine ------------------------------------------------------
    def combine(self, route: Route, resid: torch.Tensor | None = None, out: torch.Tensor | None = None,
                stream=None) -> torch.Tensor:
        m = self.g.model
        if out is None:
            out = torch.empty((route.T, m.hidden), dtype=torch.bfloat16, device=self.g.device)
        _lib.call("msi_combine", self.g.ctx, ops._ptr(out), ops._ptr(route.w), ops._ptr(route.dest),
                  ops._ptr(route.slot), ops._ptr(resid), route.T, route.mb, route.epoch, ops._stream(stream))
        return out

    def gather_y(self, route: Route, stream=None) -> torch.Tensor:
        """The expert outputs of the route's rows, [T, K, H] (with expert TP
        [T, K, tp, H]): what the combine pulled (verification; call after
        the combine of the same micro-batch)."""
        m, tp = self.g.model, self.g.plan.tp_e
        shape = (route.T, m.topk, m.hidden) if tp == 1 else (route.T, m.topk, tp, m.hidden)
        y = torch.empty(shape, dtype=torch.bfloat16, device=self.g.device)
        _lib.call("msi_gather_y", self.g.ctx, ops._ptr(y), ops._ptr(route.dest), ops._ptr(route.slot), route.T,
                  route.mb, ops._stream(stream))
        return y


# ------------------------------------------------------------- pipeline -----
PHASES = ("attn", "disp", "ffn", "comb")


class PingPongRunner:
    """m micro-batches x L layers.

    Attention GPU program order (FIFO, the schedule SPEC.md:264-272 simulates):
      for i in range(m*L): j, l = i % m, i // m
          if l > 0: comb(j, l-1)      # waits for the expert GPUs' epoch
          attn(j, l); router(j, l); disp(j, l)
      comb(j, L-1) for all j
    Expert GPU: for l: for j: ffn(j, l)      (waits for all senders' epoch)
    Co-located GPU: for l: for j: attn, router, disp, ffn, comb.
    Residual: x_{l+1} = x_l + MoE(x_l), written in place by the combine.
    """

    def __init__(self, layer: MoEDecodeLayer, layers: int, record_timeline: bool = False,
                 chain: bool = True, attn: list | None = None):
        self.layer = layer
        self.L = layers
        g = layer.g
        # attn: one attention.AttentionStage per micro-batch (attention ranks):
        # the real decode attention layer whose output feeds the MoE layer.
        # Without it the MoE layer reads x directly.
        self.attn = attn if g.is_attention else None
        if self.attn is not None and len(self.attn) != g.plan.m:
            raise ValueError("need one AttentionStage per micro-batch")
        # chain=False: every layer reads the same x and writes x + MoE(x) to a
        # separate buffer (benchmarks: random-init SwiGLU layers without a norm
        # grow |x| quadratically and overflow when chained; the cross-GPU
        # dependencies and work per layer are unchanged).
        self.chain = chain
        self.outs = None
        if not chain and g.is_attention:
            self.outs = [torch.empty((g.plan.b_a, g.model.hidden), dtype=torch.bfloat16, device=g.device)
                         for _ in range(g.plan.m)]
        self.record = record_timeline
        self.events = []
        self.fused = os.environ.get("MSI_FUSED_DISPATCH", "1") != "0"

    def _attn(self, j, l, x):
        """Attention stage of micro-batch j, layer l -> the MoE layer's input."""
        if self.attn is not None:
            return self.attn[j].forward(x, l)
        return x

    def _route_dispatch(self, h, j):
        """Router + M2N dispatch of micro-batch j: one fused launch by default
        (MSI_FUSED_DISPATCH=0: router and dispatch kernels, for A/B runs)."""
        lay = self.layer
        if self.fused:
            return lay.route_dispatch(h, j)
        r = lay.router(h, j)
        lay.dispatch(h, r, j)
        return r

    def _out(self, xs, j):
        return xs[j] if self.chain else self.outs[j][: xs[j].shape[0]]

    def _ev(self, tag):
        if self.record:
            # external: inside a CUDA-graph capture the record becomes a graph
            # node, so every replay re-stamps it (read after the last replay)
            e = torch.cuda.Event(enable_timing=True, external=True)
            e.record()
            self.events.append((tag, e))

    def run(self, xs: list | None):
        """xs: m token tensors [b_a, H] bf16 (attention ranks; updated in place)."""
        lay, g = self.layer, self.layer.g
        m, L = g.plan.m, self.L
        self.events = []
        if g.role == "both":
            for l in range(L):
                for j in range(m):
                    self._ev(("attn", j, l, 0)); h = self._attn(j, l, xs[j]); self._ev(("attn", j, l, 1))
                    self._ev(("disp", j, l, 0))
                    r = self._route_dispatch(h, j)
                    self._ev(("disp", j, l, 1))
                    lay.expert_wait(j); self._ev(("ffn", j, l, 0)); lay.expert_ffn(j); self._ev(("ffn", j, l, 1))
                    self._ev(("comb", j, l, 0)); lay.combine(r, resid=h, out=self._out(xs, j)); self._ev(("comb", j, l, 1))
        elif g.role == "attention":
            routes, hs = [None] * m, [None] * m
            for i in range(m * L):
                j, l = i % m, i // m
                if l > 0:
                    self._ev(("comb", j, l - 1, 0))
                    lay.combine(routes[j], resid=hs[j], out=self._out(xs, j))
                    self._ev(("comb", j, l - 1, 1))
                self._ev(("attn", j, l, 0)); hs[j] = self._attn(j, l, xs[j]); self._ev(("attn", j, l, 1))
                self._ev(("disp", j, l, 0))
                routes[j] = self._route_dispatch(hs[j], j)
                self._ev(("disp", j, l, 1))
            for j in range(m):
                self._ev(("comb", j, L - 1, 0))
                lay.combine(routes[j], resid=hs[j], out=self._out(xs, j))
                self._ev(("comb", j, L - 1, 1))
        else:
            for l in range(L):
                for j in range(m):
                    lay.expert_wait(j); self._ev(("ffn", j, l, 0)); lay.expert_ffn(j); self._ev(("ffn", j, l, 1))
        return xs

    # -- CUDA graph: one whole step (m x L) captured per rank -----------------
    def capture(self, xs: list | None):
        """Capture one step into a CUDA graph.  Epochs switch to device-tracked
        mode (epoch 0 in the ABI), so every replay is the next use of each slot
        and peers stay in lock-step through their own graphs' device waits."""
        self.layer.device_epochs = True
        side = torch.cuda.Stream(device=self.layer.g.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.run(xs)  # eager step in device-epoch mode (first-use attribute setup)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=side):
            self.run(xs)
        torch.cuda.synchronize()
        return self.graph

    def replay(self):
        self.graph.replay()

    def timeline(self):
        """Per-phase (phase, mb, layer, start_ms, end_ms) relative to the first
        event (call after synchronize)."""
        if not self.events:
            return []
        t0 = self.events[0][1]
        opened = {}
        rows = []
        for (ph, j, l, edge), ev in self.events:
            if edge == 0:
                opened[(ph, j, l)] = ev
            else:
                s = opened.pop((ph, j, l))
                rows.append((ph, j, l, t0.elapsed_time(s), t0.elapsed_time(ev)))
        return rows

    def stage_times_ms(self) -> dict:
        """Median per-(micro-batch, layer) duration of each phase (ms) from the
        last recorded step: attention-side work T_a = attn + disp (router and
        M2N send run on the attention GPU's SMs), expert T_e = ffn (both GEMMs,
        N2M send in the GEMM2 epilogue), comb = the combine kernel including
        its wait for the expert GPUs."""
        import statistics

        per = {}
        for ph, j, l, s, e in self.timeline():
            per.setdefault(ph, {})[(j, l)] = e - s
        out = {ph: statistics.median(v.values()) for ph, v in per.items()}
        if "attn" in per or "disp" in per:
            keys = set(per.get("attn", {})) | set(per.get("disp", {}))
            out["T_a"] = statistics.median(per.get("attn", {}).get(k, 0.0) + per.get("disp", {}).get(k, 0.0)
                                           for k in keys)
        if "ffn" in per:
            out["T_e"] = out["ffn"]
        return out


def synth_device_weights(model: MoeModelSpec, experts, seed: int = 0, device="cuda", tp: int = 1,
                         tp_rank: int = 0):
    """Random-init bf16 weights on the device (SURVEY.md §8(d) scales):
    wg ~ N(0, 1/H), W_gate/W_up ~ N(0, 1/H), W_down ~ N(0, 1/H').  Returns
    (wg [E,H], w13 [E_l,2H'/tp,H] packed, w2 [E_l,H,H'/tp]); with expert TP
    the slice of features [tp_rank H'/tp, (tp_rank+1) H'/tp) of every expert."""
    H, Hp, E = model.hidden, model.intermediate, model.experts
    Hs = Hp // tp
    f0 = tp_rank * Hs
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    wg = (torch.randn((E, H), generator=gen, device=device) / H ** 0.5).to(torch.bfloat16)
    experts = list(experts)
    w13 = torch.empty((len(experts), 2 * Hs, H), dtype=torch.bfloat16, device=device)
    w2 = torch.empty((len(experts), H, Hs), dtype=torch.bfloat16, device=device)
    for i, e in enumerate(experts):
        if e < 0:  # empty slot of a replicated placement: never routed to
            w13[i].zero_()
            w2[i].zero_()
            continue
        gen.manual_seed(seed * 100003 + 1 + e)
        wgt = (torch.randn((1, Hp, H), generator=gen, device=device) / H ** 0.5).to(torch.bfloat16)
        wup = (torch.randn((1, Hp, H), generator=gen, device=device) / H ** 0.5).to(torch.bfloat16)
        w13[i:i + 1] = ops.pack_w13(wgt[:, f0:f0 + Hs].contiguous(), wup[:, f0:f0 + Hs].contiguous())
        del wgt, wup
        w2[i] = (torch.randn((H, Hp), generator=gen, device=device) / Hp ** 0.5).to(torch.bfloat16)[:, f0:f0 + Hs]
    return wg, w13, w2


def local_experts(group: M2NGroup) -> list:
    """Logical expert behind each local (physical) slot of this expert GPU, in
    slot order; -1 marks an empty slot of a replicated placement."""
    if not group.is_expert:
        return []
    if group.slots is not None:
        return group.slots.logical_of_local(group.expert_index)
    return list(range(group.node * group.E_l, (group.node + 1) * group.E_l))


def init_distributed_from_env(backend: str = "nccl"):
    """torchrun-style init (RANK/WORLD_SIZE/LOCAL_RANK, MASTER_ADDR=127.0.0.1)."""
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if os.environ.get("MSI_OVERSUBSCRIBE") == "1" and torch.cuda.is_available():
        local %= torch.cuda.device_count()  # validation runs: several ranks per GPU (use gloo)
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group(backend, rank=rank, world_size=world,
                                device_id=torch.device(f"cuda:{local}") if backend == "nccl" else None)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local
