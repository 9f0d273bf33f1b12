#!/usr/bin/env python
"""Decode-step benchmark: disaggregated-EP MoE layer with ping-pong micro-batches.

Metric (BASELINE.json): "decode tokens/s/GPU (MoE layer, ping-pong); M2N
dispatch+combine p50 us".  One step = one decode iteration of the MoE layer
over L_sim layers (one layer's weights reused) for m
micro-batches of b_a tokens per attention GPU, on synthetic random-init
weights and activations.  ``value`` = whole-job layer-tokens/s
= n_a * m * b_a * L_sim / step time (``value_per_gpu`` divides by N).

Workloads (config 3 of BASELINE.json, Mixtral-8x22B-shaped, b_a = 1024, m = 3):
  N=1 co-located (both roles on one GPU, M2N local); N=2 1+1; N=4 3+1; N=8 6+2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

# --impl reference under torchrun (N > 1): torchrun pins OMP_NUM_THREADS=1 in
# every rank, which would leave rank 0's CPU arm on one core.  Give it the
# host threads before numpy / OpenBLAS / the OpenMP oracle read the variable.
_argv = " ".join(sys.argv[1:])
if os.environ.get("WORLD_SIZE", "1") != "1" and ("--impl reference" in _argv or "--impl=reference" in _argv):
    _n = str(len(os.sched_getaffinity(0)))
    for _k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[_k] = _n

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SPLITS = {1: (1, 1, True), 2: (1, 1, False), 4: (3, 1, False), 8: (6, 2, False),
          3: (2, 1, False), 5: (4, 1, False), 6: (4, 2, False), 7: (5, 2, False)}


def apply_plan_json(args):
    """--plan-json: the planner's DeploymentPlan (and model) replace the layout,
    m and b_a arguments; returns the fixed (n_a, n_e, colocated, source, tp_e)."""
    from paper_2504_02263_b200.config import load_plan
    bundle, plan = load_plan(args.plan_json)
    args.shape = bundle.model
    args.m, args.b_a = plan.m, plan.b_a
    args.tp_a = plan.tp_a  # attention nodes of tp_a GPUs
    return plan.n_a, plan.n_e, plan.colocated, f"--plan-json {os.path.basename(args.plan_json)}", plan.tp_e


def choose_split(world: int, shape: str, plan_arg: str, split: str = "", colocated: bool = False,
                 tp_e: int = 1):
    """(n_a, n_e expert GPUs, colocated, source, tp_e) for this run.

    --split a+e / --colocated force a layout.  --plan config uses the
    BASELINE.json configuration splits (SPLITS: 1+1, 3+1, 6+2 ...).  The
    default, --plan planner, asks Algorithm 1 (planner.search_box)
    for the best layout of this box with the B200-calibrated coefficients of
    profiles/r01_calibration_<shape>.json; shapes without a calibration fall
    back to the config splits.  For Mixtral-8x22B the search picks co-location
    at every N > 1 (the disaggregated splits fail its balance constraint:
    T_a is ~half of T_e per token on identical GPUs)."""
    if split:
        n_a, n_e = (int(v) for v in split.split("+"))
        if n_a + n_e != world:
            raise SystemExit(f"--split {split} needs {n_a + n_e} GPUs")
        return n_a, n_e, False, "--split", tp_e
    if colocated or world == 1:
        return world, world, True, "--colocated" if colocated else "1 GPU: co-located", 1
    if plan_arg == "planner":
        import glob
        cal, cal_path = None, ""
        for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_calibration_*.json"))):
            with open(path) as fh:
                c = json.load(fh)
            if str(c.get("shape", "")).lower() == shape.lower():
                cal, cal_path = c, os.path.relpath(path, ROOT)
        if cal is not None:
            from paper_2504_02263_b200 import perf_model as PM
            from paper_2504_02263_b200 import planner as PL
            from paper_2504_02263_b200.config import WorkloadSpec, as_model_spec, b200_gpu
            c = cal
            cm = PM.CostModel(k1=c["k1_s_per_tok"], k2=c["k2_s"], k3=c["k3_s_per_tok"], k4=c["k4_s"],
                              util_curve=PM.UtilCurve.from_points(c["util_table"]))
            p = PL.search_box(as_model_spec(shape), b200_gpu(), PL.cm_scaled_for_experts(cm, c["experts_local"]),
                              WorkloadSpec(), world)
            if p:
                src = f"planner.search_box (calibrated B200 costs, {cal_path})"
                if p.tp_e > 1:  # expert nodes of tp_e GPUs
                    src += f"; expert TP {p.tp_e}"
                if p.tp_a > 1:  # attention nodes of tp_a GPUs: the runtime counts attention GPUs
                    src += f"; attention TP {p.tp_a} (use --tp-a {p.tp_a})"
                return p.n_a * p.tp_a, p.n_e * p.tp_e, bool(p.colocated), src, p.tp_e
    n_a, n_e, colo = SPLITS[world]
    return n_a, n_e, colo, "BASELINE.json config split", tp_e


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--shape", default="mixtral-8x22b")
    ap.add_argument("--b-a", type=int, default=1024)
    # (not "--m": torchrun would take it as an abbreviation of its own options)
    ap.add_argument("--micro-batches", dest="m", type=int, default=3, help="m, micro-batches per step")
    ap.add_argument("--layers", type=int, default=4, help="L_sim layers per step")
    ap.add_argument("--attn", default="real", choices=["real", "none"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--split", default="", help="attention+expert GPUs, e.g. 6+2 (disaggregated)")
    ap.add_argument("--tp-a", dest="tp_a", type=int, default=1,
                    help="attention GPUs per attention node (tensor parallel over heads; all-gather/reduce-scatter "
                         "fused into the projection GEMMs)")
    ap.add_argument("--tp-e", dest="tp_e", type=int, default=1,
                    help="expert GPUs per expert node (tensor parallel over h'; disaggregated layouts)")
    ap.add_argument("--plan-json", default="", help="a planner output (python -m paper_2504_02263_b200.planner "
                    "--out ...): model, layout, m and b_a from its plan section")
    ap.add_argument("--plan", default="planner", choices=["planner", "config"],
                    help="N > 1 layout: Algorithm 1 on the calibrated B200 costs (default) or the BASELINE config splits")
    ap.add_argument("--skew", type=float, default=0.0,
                    help="make experts 0/1 hot (gate-logit bias); 0 = random-init routing")
    ap.add_argument("--balance", action="store_true",
                    help="replicate hot experts across expert GPUs (balance_experts, SPEC.md:407-414)")
    ap.add_argument("--timeline-csv", default="",
                    help="write the SPEC timeline CSV of the last timed step ('{rank}' is substituted)")
    ap.add_argument("--colocated", action="store_true",
                    help="every GPU is both an attention and an expert GPU (DeepSeek-V3-shaped config 5)")
    ap.add_argument("--no-merge", dest="merge", action="store_false",
                    help="co-located layouts (any N): keep m separate micro-batches instead of one merged batch")
    ap.add_argument("--no-pingpong", dest="pingpong", action="store_false",
                    help="N > 1 co-located headline: skip the secondary disaggregated ping-pong measurement")
    ap.add_argument("--no-m2n", action="store_true", help="skip the M2N round-trip p50 measurement")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch eagerly from Python instead of replaying a captured CUDA graph")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled DURING the timed
    region: NVML polled every 5 ms on a thread; only samples between
    window_open() and window_close() (wall clock around the timed loop and
    its final synchronize) count.  Falls back to nvidia-smi -lms 100 when
    NVML is unavailable."""

    NAMES = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
             ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (t, sm_mhz, reasons_mask, power_w)
        self.smax = None
        self.win = [None, None]
        self._stop = threading.Event()
        self.t = None
        self.nv = None

    def _handle(self):
        import pynvml as nv
        nv.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            h = nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
        return nv, h

    def start(self):
        try:
            self.nv, self.h = self._handle()
            self.smax = float(self.nv.nvmlDeviceGetMaxClockInfo(self.h, self.nv.NVML_CLOCK_SM))
        except Exception:
            self.nv = None
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv, h = self.nv, self.h
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1e3
                self.samples.append((time.perf_counter(), float(sm), int(rs), pw))
            except Exception:
                pass
            time.sleep(0.005)

    def window_open(self):
        self.win[0] = time.perf_counter()

    def window_close(self):
        self.win[1] = time.perf_counter()

    def stop(self) -> dict:
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self._stop.set()
        self.t.join(timeout=1)
        t0, t1 = self.win
        inside = [x for x in self.samples if t0 is not None and t1 is not None and t0 <= x[0] <= t1]
        sm = [x[1] for x in inside]
        reasons = set()
        for x in inside:
            for n, bit in self.NAMES:
                if x[2] & bit:
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                "sm_mhz_min": min(sm) if sm else None, "power_w_median": statistics.median(x[3] for x in inside)
                if inside else None, "reasons": sorted(reasons), "samples": len(sm),
                "how": "NVML every 5 ms, samples inside the timed region only"}


def ncu_traffic(name: str, b_a: int, n_a: int, n_e: int, colo: bool) -> dict | None:
    """DRAM bytes per launch of the dominant kernels from the committed ncu
    capture of this exact configuration (profiles/r02_ncu_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
    if not os.path.exists(path):
        return None
    key = f"{name}|{b_a}|{n_a}+{n_e}|{'colo' if colo else 'disagg'}"
    return json.load(open(path)).get(key)


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


# --------------------------------------------------------------- CPU leg ----
_CPU_CACHE = {}


def cpu_layer(model, T: int, attn: bool = True, steps: int = 1, warmup: int = 0, seed: int = 0) -> dict:
    """The CPU baseline: oracle.CpuDecodeLayer (oracle/) executes the whole
    layer step for the T tokens of one attention GPU's step on the host cores
    -- attention stage over every sequence's paged KV cache (s = 730 mean),
    router + placement, every expert's SwiGLU FFN over its routed rows, combine
    -- nothing sampled or projected.  Returns the median over ``steps`` timed
    steps after ``warmup`` untimed ones."""
    from oracle import oracle as O
    from paper_2504_02263_b200.attention import ROPE_THETA, head_layout
    from paper_2504_02263_b200.config import WorkloadSpec

    key = (model.name, T, attn)
    if key not in _CPU_CACHE:  # inputs and weights are not part of the timed step
        n_heads, n_kv = head_layout(model)
        ctx = np.random.default_rng(seed + 3).integers(1, 2 * WorkloadSpec().avg_seq_len, size=T).astype(np.int32)
        lay = O.CpuDecodeLayer(model.hidden, model.intermediate, model.experts, model.topk, T, n_heads, n_kv, ctx,
                               theta=ROPE_THETA, seed=seed)
        _CPU_CACHE[key] = (lay, O.fill_normal((T, model.hidden), seed + 5))
    lay, x = _CPU_CACHE[key]
    times, phases = [], []
    for i in range(warmup + steps):
        if attn:
            _, ph = lay.step(x)
        else:
            t0 = time.perf_counter()
            lay.moe(x)
            ph = {"attention_s": 0.0, "moe_s": time.perf_counter() - t0}
            ph["layer_s"] = ph["moe_s"]
        if i >= warmup:
            times.append(ph["layer_s"])
            phases.append(ph)
    t = statistics.median(times)
    ph = phases[times.index(t)] if t in times else phases[-1]
    return {"tokens_per_s": T / t, "t_layer_s": t, "t_attention_s": ph["attention_s"], "t_moe_s": ph["moe_s"],
            "sample": (f"the whole layer step for {T} tokens per step (one attention GPU's m x b_a), no sampling: "
                       + ("attention stage (QKV projection, RoPE + paged-KV append, GQA decode over every "
                          "sequence's cache at s = 730 mean, output projection + residual), " if attn else "")
                       + f"router + placement, SwiGLU FFN of all {model.experts} experts over their routed rows, "
                       "combine; oracle/ (numpy/OpenBLAS fp32 GEMMs + OpenMP C)")}


def eq5_report(all_stages: list, plan, L: int, ms_per_step: float, colocated: bool) -> dict:
    """Measured T_a / T_e (medians over micro-batches and layers, max over the
    GPUs of a role) against the reference's closed form Eq. 5 (PAPER.md:237,
    SPEC.md:246-254): T_total = (T_a + T_e + 2 T_c) + T_f (m L - 1).  T_c is 0
    here: dispatch and the N2M send run on SMs inside T_a and T_e."""
    from paper_2504_02263_b200.pipeline import StageTimes, closed_form_total, simulate

    t_a = max((s.get("T_a", 0.0) for s in all_stages), default=0.0)
    t_e = max((s.get("T_e", 0.0) for s in all_stages), default=0.0)
    comb = max((s.get("comb", 0.0) for s in all_stages), default=0.0)
    rep = {"T_a_ms": t_a, "T_e_ms": t_e, "comb_ms": comb, "m": plan.m, "L": L, "T_c_ms": 0.0}
    if colocated:
        # both stages share one GPU: no overlap, the step is the sum
        pred = plan.m * L * (t_a + t_e + comb)
        rep.update(model="co-located sum m*L*(T_a+T_e+comb)", predicted_ms=pred)
    else:
        st = StageTimes(t_a, t_e, 0.0)
        pred = closed_form_total(st, plan.m, L)
        rep.update(model="Eq. 5 closed_form_total", predicted_ms=pred,
                   simulated_ms=simulate(st, plan.m, L).total_latency)
    rep["measured_ms"] = ms_per_step
    rep["measured_over_predicted"] = ms_per_step / pred if pred else None
    return rep


def m2n_latency(layer, g, x, world: int, iters: int = 1000, warm: int = 50) -> dict | None:
    """The metric's second half: M2N dispatch + N2M combine round trip p50/p99
    (µs) for this config's micro-batch (x = the MoE layer input of micro-batch
    0 on attention ranks), with an identity expert step (msi_expert_echo) in
    between so the expert GEMM is not counted.  One CUDA graph replay per
    iteration, barrier + synchronize around each, max over ranks
    (>= 1000 iterations after >= 50 warm-up)."""
    import torch
    import torch.distributed as dist

    route = layer.router(x, 0) if g.is_attention else None
    out = torch.empty_like(x) if g.is_attention else None

    mid = torch.cuda.Event(enable_timing=True, external=True)  # end of the dispatch leg (graph node)

    def trip():
        if g.is_attention:
            layer.dispatch(x, route, 0)
            mid.record()
        if g.is_expert:
            layer.expert_echo(0)
        if g.is_attention:
            layer.combine(route, out=out)

    for _ in range(3):
        trip()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    gr = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(device=x.device if x is not None else None)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(gr, stream=side):
        trip()
    torch.cuda.synchronize()
    lat, disp = [], []
    for i in range(warm + iters):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        gr.replay()
        e.record()
        torch.cuda.synchronize()
        if i >= warm:
            lat.append(s.elapsed_time(e) * 1e3 if g.is_attention else 0.0)
            disp.append(s.elapsed_time(mid) * 1e3 if g.is_attention else 0.0)
    t = torch.tensor(lat + disp, dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))
    if world > 1:
        allreduce_(t, dist.ReduceOp.MAX)
    tl = t.cpu().tolist()
    v = sorted(tl[:len(lat)])
    dv = sorted(tl[len(lat):])
    # steady state: CHAIN round trips back to back in one graph (a decode
    # loop's layers), so the per-iteration host-barrier skew is paid once per
    # CHAIN; per-trip time = replay time / CHAIN, max over ranks, p50
    CHAIN, reps = 16, 64
    grc = torch.cuda.CUDAGraph()
    with torch.cuda.graph(grc, stream=side):
        for _ in range(CHAIN):
            trip()
    torch.cuda.synchronize()
    chain = []
    for i in range(reps + 4):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        grc.replay()
        e.record()
        torch.cuda.synchronize()
        if i >= 4:
            chain.append(s.elapsed_time(e) * 1e3 / CHAIN if g.is_attention else 0.0)
    tc = torch.tensor(chain, dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))
    if world > 1:
        allreduce_(tc, dist.ReduceOp.MAX)
    cv = sorted(tc.cpu().tolist())
    if g.status() != 0:
        raise RuntimeError("device status after the M2N round trips")
    T, H, K = (x.shape[0], x.shape[1], g.model.topk) if x is not None else (0, 0, 0)
    p50 = v[len(v) // 2]
    c50 = cv[len(cv) // 2]
    return {"p50_us": p50, "p99_us": v[min(len(v) - 1, int(0.99 * len(v)))], "iters": iters,
            "dispatch_leg_p50_us": dv[len(dv) // 2],
            "tokens_per_attention_gpu": T, "dispatch_bytes_per_attention_gpu": T * K * H * 2,
            "how": "graph replay of dispatch -> expert echo -> combine, barrier each, max over ranks",
            "roofline": m2n_roofline(g, route, world, g.model.hidden, p50, dv[len(dv) // 2]),
            "steady_state": {"per_trip_p50_us": c50, "chain": CHAIN, "replays": reps,
                             "roofline": m2n_roofline(g, route, world, g.model.hidden, c50),
                             "how": f"{CHAIN} round trips back to back per graph replay, per-trip p50, max over ranks"}}


SM_STORE_GBS = 689.0  # measured ceiling of SM peer stores per direction, bidirectional (see m2n_roofline)


def _over() -> bool:
    """MSI_OVERSUBSCRIBE=1: validation runs with more ranks than GPUs (ranks
    share GPUs round-robin, host collectives over gloo).  Numbers from such a
    run are not measurements."""
    return os.environ.get("MSI_OVERSUBSCRIBE") == "1"


def allreduce_(t, op=None):
    """In-place all-reduce of a (device) tensor; staged through the host on gloo."""
    import torch.distributed as dist
    op = op if op is not None else dist.ReduceOp.SUM
    if dist.get_backend() == "gloo" and t.is_cuda:
        c = t.cpu()
        dist.all_reduce(c, op=op)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=op)


def allgather(t) -> list:
    import torch
    import torch.distributed as dist
    src = t.cpu() if dist.get_backend() == "gloo" else t
    out = [torch.zeros_like(src) for _ in range(dist.get_world_size())]
    dist.all_gather(out, src)
    return out


def m2n_leg_bytes(mat, H: int):
    """mat[src][dst] = (t, k) rows attention rank src routes to GPU dst.
    Returns (dispatch-leg bytes, return-leg bytes, remote-rows matrix) of the
    busiest GPU: rows a GPU keeps for itself never cross NVLink; per leg the
    bound is max over GPUs of max(egress, ingress); dispatch rows carry 8 B of
    metadata on top of the 2H-byte row, returned rows do not."""
    n = len(mat)
    off = [[0 if i == j else int(mat[i][j]) for j in range(n)] for i in range(n)]
    out_rows = [sum(r) for r in off]
    in_rows = [sum(off[i][j] for i in range(n)) for j in range(n)]
    busiest = max(max(o, i) for o, i in zip(out_rows, in_rows)) if n else 0
    return busiest * (2 * H + 8), busiest * 2 * H, off


def m2n_roofline(g, route, world: int, H: int, p50_us: float, disp_us: float | None = None) -> dict:
    """Bytes the round trip must move and the rate it reached.

    N > 1: the two legs run one after the other (rows out, rows back), so the
    link-time lower bound is, per leg, the busiest GPU's max(egress, ingress)
    NVLink bytes (dispatch: 2H + 8 B metadata per remote (t, k) row; return:
    2H), summed over the legs.  achieved = those bytes / p50, against the
    measured 770 GB/s peer copy per direction (B200_PROFILING.md) and the
    900 GB/s nominal.  N = 1: everything is local, so the bound is HBM:
    dispatch reads x and writes T*K rows, the echo reads and writes T*K rows,
    the combine reads T*K rows and writes T; against MEASURED_PEAKS hbm_gbs."""
    import torch
    import torch.distributed as dist

    dev = torch.device("cuda", torch.cuda.current_device())
    plan = g.plan
    rows_to = torch.zeros(world, dtype=torch.int64, device=dev)
    if g.is_attention and route is not None:
        node = (route.dest.to(torch.int64) // g.E_l).flatten()
        ranks = torch.tensor(plan.expert_ranks(), dtype=torch.int64, device=dev)
        for r in range(plan.tp_e):  # expert TP: every GPU of the node receives the row
            rows_to += torch.bincount(ranks[node * plan.tp_e + r], minlength=world)[:world]
    if world > 1:
        mat = torch.stack([m.cpu() for m in allgather(rows_to)])
    else:
        mat = rows_to.cpu()[None, :]
    if world == 1:
        rows = int(mat.sum())
        T = route.T if route is not None else 0
        by = T * H * 2 + rows * H * 2 + 2 * rows * H * 2 + rows * H * 2 + T * H * 2
        peak = measured_peaks().get("hbm_gbs") or 6546.6
        gbs = by / (p50_us * 1e-6) / 1e9
        return {"bound": "hbm", "bytes": by, "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                "peak_kind": "measured hbm_gbs (MEASURED_PEAKS.json); co-located 1 GPU: all rows local"}
    leg1, leg2, off = m2n_leg_bytes(mat.tolist(), H)
    by = leg1 + leg2
    gbs = by / (p50_us * 1e-6) / 1e9
    dl = None
    if disp_us:  # the dispatch leg alone (its kernel's end event; includes the count exchange)
        a = leg1 / (disp_us * 1e-6) / 1e9
        dl = {"p50_us": disp_us, "achieved": a, "frac": a / 770.0, "frac_nominal": a / 900.0,
              "frac_sm_store_ceiling": a / SM_STORE_GBS}
    return {"bound": "nvlink", "bytes_busiest_gpu": by, "dispatch_leg_bytes": leg1, "return_leg_bytes": leg2,
            "dispatch_leg": dl,
            "remote_rows_matrix": off, "achieved": gbs, "unit": "GB/s",
            "peak": 770.0, "frac": gbs / 770.0, "peak_kind": "measured peer copy per direction (B200_PROFILING.md)",
            "nominal": 900.0, "frac_nominal": gbs / 900.0,
            # SM-issued 16-B peer stores saturate below the copy engines on this
            # pool: 689 GB/s per direction both ways at once, 695 one way
            # (scripts/peer_store_probe.cu, profiles/r01_peer_store_probe.jsonl)
            "sm_store_ceiling": SM_STORE_GBS, "frac_sm_store_ceiling": gbs / SM_STORE_GBS}


def cpu_model_name() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _u16(t) -> "np.ndarray":
    return t.detach().contiguous().view(__import__("torch").int16).cpu().numpy().view(np.uint16)


def parity_check(layer, g, runner, att_stages, xs, wg, w13, w2, model, n_experts_checked: int = 2) -> dict | None:
    """Oracle parity of the bench's own data, outside the timed region: the
    MoE input of micro-batch 0 at the last layer of the last timed step (the
    attention stage's output) and what the GPU made of it.  Routing (idx, w,
    cnt, slot) must be bit-exact; the combine is bit-exact
    given the GPU's expert outputs; on a rank that holds every expert (N = 1)
    the outputs of ``n_experts_checked`` experts are compared with the
    oracle's SwiGLU within the bf16 tolerance (rel-L2 <= 5e-3, max-abs <=
    2^-7 max|ref|).  Returns None on ranks without the attention role."""
    from oracle import oracle as O

    if not g.is_attention:
        return None
    r = layer._routes[0]
    T, K = r.T, model.topk
    h = att_stages[0].y[:T] if att_stages else xs[0][:T]
    hx = _u16(h)
    idx_r, w_r = O.router(hx, _u16(wg), K)
    dest_r = idx_r if g.slots is None else O.physical_slots(idx_r, g.slots.rep, g.attn_index)
    cnt_r, slot_r = O.place(dest_r, g.P)
    rep = {"checked_on": "micro-batch 0, last layer of the last timed step (outside the timed region)",
           "tokens": T,
           "routing_bit_exact": bool(np.array_equal(r.idx[:T].cpu().numpy(), idx_r)
                                     and np.array_equal(r.w[:T].cpu().numpy().view(np.uint32), w_r.view(np.uint32))
                                     and np.array_equal(r.dest[:T].cpu().numpy(), dest_r)
                                     and np.array_equal(r.cnt.cpu().numpy(), cnt_r)
                                     and np.array_equal(r.slot[:T].cpu().numpy(), slot_r))}
    tp = g.plan.tp_e
    ybuf = _u16(layer.gather_y(r))
    yk = ybuf.reshape(T, K * tp, model.hidden)
    out = _u16(runner._out([x for x in xs], 0)[:T]) if xs else None
    if out is not None:
        rep["combine_bit_exact"] = bool(np.array_equal(out, O.combine(yk, np.repeat(w_r, tp, axis=1), hx)))
    if g.is_expert and g.plan.n_e == 1 and tp == 1 and g.slots is None and w13 is not None:
        rels, ok = {}, True
        loads = np.bincount(idx_r.ravel(), minlength=model.experts)
        for e in sorted({int(np.argmax(loads)), int(np.argmin(loads))} | {0})[:n_experts_checked]:
            t, k = np.nonzero(idx_r == e)
            order = np.argsort(slot_r[t, k])
            t, k = t[order], k[order]
            two_hp = w13.shape[1]
            v = w13[e].view(two_hp // 256, 2, 2, 64, model.hidden)  # msi_pack_w13 layout -> gate / up
            gate, up = _u16(v[:, :, 0].reshape(two_hp // 2, -1)), _u16(v[:, :, 1].reshape(two_hp // 2, -1))
            ref = O.bf16_to_f32(O.expert_ffn(hx[t], gate, up, _u16(w2[e]))).astype(np.float64)
            got = O.bf16_to_f32(ybuf[t, k]).astype(np.float64)
            rel = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
            mx = float(np.abs(got - ref).max()) / max(float(np.abs(ref).max()), 1e-30)
            rels[int(e)] = {"rows": int(len(t)), "rel_l2": rel, "max_abs_over_max_ref": mx}
            ok &= rel <= 5e-3 and mx <= 2.0 ** -7
        rep["experts"] = rels
        rep["experts_within_tolerance"] = bool(ok)
    return rep


def resolve_layout(args, world: int):
    """(n_a, n_e, colocated, plan_source, tp_e, model, m, b_a) of this run --
    shared by both arms so they describe the same workload."""
    from paper_2504_02263_b200.config import as_model_spec

    if args.plan_json:
        n_a, n_e, colo, plan_source, tp_e = apply_plan_json(args)
        if (n_a if colo else n_a + n_e) != world:
            raise SystemExit(f"--plan-json needs {n_a if colo else n_a + n_e} ranks, WORLD_SIZE={world}")
    else:
        n_a, n_e, colo, plan_source, tp_e = choose_split(world, args.shape, args.plan, args.split,
                                                         args.colocated, args.tp_e)
    model = as_model_spec(args.shape)
    m_eff, b_a = args.m, args.b_a
    if colo and args.merge:
        # A co-located GPU runs attention and experts on the same SMs, so a
        # ping-pong partner would only halve its GEMMs: its m micro-batches are
        # merged into one batch (same tokens per step, expert weights streamed
        # once per layer instead of m times; DESIGN.md §6 overlap probe).
        m_eff, b_a = 1, args.m * args.b_a
    return n_a, n_e, colo, plan_source, (1 if colo else tp_e), model, m_eff, b_a


def router_launch_count(E: int, T: int) -> int:
    """Launches of one router (+ dispatch) call (router.cu's path choice):
    tensor-core logits for E % 256 == 0 at T >= 1024 (expert norms, logits
    GEMM, route), the split path for E >= 64 at T <= 256 (logits, route),
    else the fused kernel."""
    env = os.environ.get("MSI_ROUTER_TC")
    if E % 256 == 0 and E <= 512 and (env == "1" or (env is None and T >= 1024)):
        return 3
    return 2 if (E >= 64 and E % 8 == 0 and T <= 256) else 1


def args_tp_a(args) -> int:
    return int(getattr(args, "tp_a", 1) or 1)


def bench_config(args, model, n_a: int, n_e: int, colo: bool, plan_source: str, tp_e: int, m: int, b_a: int,
                 world: int) -> dict:
    """The workload the line describes (identical in both arms' lines)."""
    return {"workload": f"{model.name}-shaped MoE layer, " +
            (f"co-located {world} GPU" + ("s (every GPU both roles, M2N all-to-all)" if world > 1 else "")
             if colo else f"{n_a} attention + {n_e} expert GPUs"),
            "plan_source": plan_source,
            "hidden": model.hidden, "intermediate": model.intermediate, "experts": model.experts,
            "topk": model.topk, "n_a": n_a, "n_e": n_e, "m": m, "b_a": b_a,
            "tokens_per_step_per_attention_gpu": m * b_a * args.layers,
            "microbatching": ("co-located: m micro-batches merged into one batch (no ping-pong partner)"
                              if colo and args.merge else "ping-pong, m micro-batches"),
            "L_sim": args.layers, "attention_stage": args.attn,
            "attention_batches": ("uniform context lengths (mean 730)" if n_a == 1 else
                                  "compose_attention_batches over the attention GPUs (SPEC.md:415-423; "
                                  "uniform request lengths, mean 730)"),
            "l2": (f"working set (expert weights {model.experts * 3 * model.hidden * model.intermediate * 2 / 1e9:.1f} GB"
                   " + KV cache) >> 126 MB L2; no flush needed"),
            "parallelism": (f"dp{n_a // args_tp_a(args)}-atp{args_tp_a(args)}" if args_tp_a(args) > 1 else f"dp{n_a}")
                           + f"-ep{n_e}" + (f"-etp{tp_e}" if tp_e > 1 else ""),
            "tp_a": args_tp_a(args),
            "launch": "CUDA graph per rank (device-tracked epochs)" if args.graph else "eager"}


def run_reference(args):
    """--impl reference: the reference ships no implementation of this path
    (SURVEY.md §0), so its CPU restatement (oracle/, kind "port") runs the
    same workload on the host cores: each step is the whole layer for one
    attention GPU's m x b_a tokens (attention stage, router, all experts,
    combine; nothing projected).  ``value`` is the host's layer-tokens/s --
    a CPU throughput, not a per-GPU figure.  Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = args.gpus
    n_a, n_e, colo, plan_source, tp_e, model, m_eff, b_a = resolve_layout(args, world)
    threads = len(os.sched_getaffinity(0))
    T = m_eff * b_a  # tokens of one attention GPU per layer step
    attn = args.attn == "real"
    cpu_layer(model, T, attn=attn, steps=1, warmup=0)  # build weights / KV cache (untimed setup) + first touch
    secs = []
    info = None
    t_all = time.perf_counter()
    for i in range(args.warmup + args.steps):
        info = cpu_layer(model, T, attn=attn, steps=1, warmup=0)
        if i >= args.warmup:
            secs.append(info["t_layer_s"])
    v = T * len(secs) / sum(secs)
    line = {"impl": "reference", "metric": "decode tokens/s/GPU (MoE layer, ping-pong); M2N dispatch+combine p50 µs",
            "value": v, "unit": "layer-tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(secs) / len(secs), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, N(0,1) tokens)",
            "config": bench_config(args, model, n_a, n_e, colo, plan_source, tp_e, m_eff, b_a, world),
            "cpu_baseline": {"value": v, "unit": "layer-tokens/s", "cores": threads, "kind": "port",
                             "sample": info["sample"], "cpu": cpu_model_name(),
                             "t_attention_s": info["t_attention_s"], "t_moe_s": info["t_moe_s"],
                             "note": "host CPU throughput for one attention GPU's tokens per step; not a per-GPU "
                                     "figure (the reference has no GPU implementation of this path)"},
            "e2e": {"value": v, "unit": "layer-tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t_all}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU leg ----
def disaggregated_layout(args, world: int, expert_share: float):
    """Best disaggregated split of `world` GPUs for the ping-pong line: with
    s = T_e / (T_a + T_e) the expert share of the measured per-token GPU time,
    n_a attention and n_e expert GPUs sustain min(n_a / (1 - s), n_e / s)
    tokens per unit time (the slower stage bounds the pipeline);
    n_e in [1, world - 1] maximises it (rounding world * s instead picks 1+3
    over 2+2 at s = 0.63, measured 1.39 M vs 1.59 M layer-tokens/s),
    m = --micro-batches separate micro-batches of --b-a tokens per attention
    GPU.  When n_e does not divide E the experts are spread over slots
    (balance.spread_slots: whole experts plus replicas of the remainder on
    every expert GPU)."""
    from paper_2504_02263_b200.balance import spread_slots
    from paper_2504_02263_b200.config import as_model_spec

    model = as_model_spec(args.shape)
    s = min(max(expert_share, 1e-6), 1 - 1e-6)
    n_e = max(range(1, world), key=lambda n: (min((world - n) / (1 - s), n / s), -n)) if world > 1 else 1
    n_a = world - n_e
    slots = spread_slots(model.experts, n_e) if model.experts % n_e else None
    src = (f"disaggregated {n_a}+{n_e}: n_e maximises min(n_a/(1-s), n_e/s), s = T_e/(T_a+T_e) = "
           f"{expert_share:.3f} from the co-located headline's stage times"
           + (f"; {slots.P} expert slots (spread_slots)" if slots else ""))
    return (n_a, n_e, False, src, 1, model, args.m, args.b_a), slots


def pingpong_summary(sub: dict | None, expert_share: float) -> dict | None:
    """The secondary (disaggregated ping-pong) line, reduced to what compares
    with the headline."""
    if sub is None:
        return None
    keep = ("value", "value_per_gpu", "ms_per_step", "stage_times", "clocks", "gpu_launches", "attention")
    out = {k: sub.get(k) for k in keep}
    out["config"] = sub["config"]
    out["expert_share"] = expert_share
    rf = sub.get("roofline") or {}
    out["expert_ffn"] = {k: rf.get(k) for k in ("achieved", "frac", "frac_sustained", "avg_launch_pair_ms", "unit")}
    par = sub.get("parity") or {}
    out["parity"] = {"routing_bit_exact": par.get("routing_bit_exact"),
                     "combine_bit_exact": par.get("combine_bit_exact")}
    return out


def measure(args, rank: int, world: int, local: int, layout, full: bool = True, slots_override=None):
    """Set up one layout, run the warm-up and the K timed steps, and return
    rank 0's JSON line (None on other ranks).  full=False (the secondary
    ping-pong measurement) skips the e2e, M2N latency and CPU legs."""
    import torch
    import torch.distributed as dist

    from paper_2504_02263_b200 import runtime
    from paper_2504_02263_b200.config import DeploymentPlan, WorkloadSpec

    n_a, n_e, colo, plan_source, tp_e, model, m_eff, b_a = layout
    args.b_a = b_a
    tp_a = getattr(args, "tp_a", 1) or 1
    plan = DeploymentPlan(n_a=n_a, n_e=n_e, m=m_eff, b_a=b_a, colocated=colo, tp_e=tp_e, tp_a=tp_a)
    if tp_a > 1 and (args.balance or args.skew > 0):
        raise SystemExit("--tp-a > 1 with --balance/--skew is not supported")
    dev = torch.device(f"cuda:{local}")
    gen = torch.Generator(device=dev)
    gen.manual_seed(1 + rank)
    is_attn_rank = rank in plan.attention_ranks()
    wg = runtime.synth_device_weights(model, [], seed=0, device=dev)[0]
    xs = [torch.randn((args.b_a, model.hidden), generator=gen, device=dev) for _ in range(plan.m)] if is_attn_rank else None
    if args.skew > 0:
        # hot experts: tokens share a direction u that the gate rows of experts
        # 0 and 1 favour (logit bias ~ skew), the way real routing concentrates
        gu = torch.Generator(device=dev)
        gu.manual_seed(12345)
        u = torch.randn(model.hidden, generator=gu, device=dev)
        u = u / u.norm()
        wgf = wg.float()
        # tokens share a component a*sqrt(H)*u (a = 0.3); experts 0 and 1 get
        # logit shifts of skew and 0.6*skew along it (skew 0.5 -> max/mean load ~2)
        a = 0.3
        wgf[0] += args.skew * u / (a * model.hidden ** 0.5)
        wgf[1] += 0.6 * args.skew * u / (a * model.hidden ** 0.5)
        wg = wgf.to(torch.bfloat16)
        if xs:
            xs = [x + a * u * model.hidden ** 0.5 for x in xs]
    if xs:
        xs = [x.to(torch.bfloat16) for x in xs]
    wl = WorkloadSpec()
    att_stages = None
    if args.attn == "real" and is_attn_rank and tp_a == 1:
        # real decode attention layer per micro-batch (paged KV at s = avg_seq_len)
        from paper_2504_02263_b200 import attention as attn_mod
        w_att = attn_mod.AttentionWeights(model, dev, seed=0)
        ctx = [None] * plan.m
        if n_a > 1:
            # the micro-batch's n_a * b_a requests composed over the attention
            # GPUs for equal predicted attention time
            ai = plan.attention_ranks().index(rank)
            ctx = [attn_mod.composed_ctx_lens(model, n_a, args.b_a, wl.avg_seq_len, seed=j)[0][ai]
                   for j in range(plan.m)]
        att_stages = [attn_mod.AttentionStage(model, args.b_a, args.layers, dev, weights=w_att, ctx_lens=ctx[j],
                                              avg_seq_len=wl.avg_seq_len, seed=1000 * rank + j)
                      for j in range(plan.m)]
    slots, loads = slots_override, None
    if args.balance or args.skew > 0:
        # calibration: this step's routing counts (all attention ranks), placement
        # by balance_experts(mode="replicated"), agreed by all ranks
        cnt = torch.zeros(model.experts, dtype=torch.float64, device=dev)
        if xs:
            from paper_2504_02263_b200 import ops as _ops
            for j, x in enumerate(xs):  # routing of the MoE layer input (after attention)
                h = att_stages[j].forward(x, 0) if att_stages else x
                cnt += _ops.gate_topk(h, wg, model.topk)[2].double()
        if world > 1:
            allreduce_(cnt)
        loads = cnt.cpu().numpy()
        if args.balance:
            from paper_2504_02263_b200.balance import balanced_slots
            slots = balanced_slots(loads, n_e, max_replicas=min(n_e, 2))
    g = runtime.M2NGroup(model, plan, rank=rank, device=dev, slots=slots)
    if args.attn == "real" and is_attn_rank and tp_a > 1:
        # attention nodes of tp_a GPUs: heads split, all-gather fused into the
        # QKV GEMM, reduce-scatter into the O projection (attn_tp.cu); the
        # node's tp_a * b_a requests composed over the attention nodes
        from paper_2504_02263_b200 import attention as attn_mod
        w_att = attn_mod.AttentionWeights(model, dev, seed=0)
        node = g.attn_index // tp_a
        att_stages = [attn_mod.AttentionTPStage(
            model, args.b_a, args.layers, g, j, w_att,
            attn_mod.composed_ctx_lens(model, n_a // tp_a, tp_a * args.b_a, wl.avg_seq_len, seed=j)[0][node],
            seed=1000 * node + j) for j in range(plan.m)]
    _, w13, w2 = runtime.synth_device_weights(model, runtime.local_experts(g), seed=0, device=dev, tp=g.tp,
                                              tp_rank=g.tp_rank)
    layer = runtime.MoEDecodeLayer(g, wg=wg if g.is_attention else None,
                                   w13=w13 if g.is_expert else None, w2=w2 if g.is_expert else None)
    runner = runtime.PingPongRunner(layer, layers=args.layers, chain=False,
                                    record_timeline=True, attn=att_stages)
    x0 = [x.clone() for x in xs] if xs else None

    def barrier():
        if world > 1:
            dist.barrier()

    # expert-FFN timing inside the timed region (events on the launching stream)
    ffn_events = []
    orig_ffn = layer.expert_ffn

    def timed_expert_ffn(mb=0, stream=None):
        # the runner calls expert_wait first, so these events time the FFN
        # kernels (GEMM1 + GEMM2) only, not the wait for the senders' rows
        s, e = torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True)
        s.record()
        r = orig_ffn(mb, stream)
        e.record()
        ffn_events.append((s, e))
        return r

    barrier()  # every rank set up (weights, KV cache) before the first cross-GPU wait
    for _ in range(args.warmup):
        runner.run(xs)
    torch.cuda.synchronize()
    barrier()
    # The step is captured once into a CUDA graph (device-tracked epochs) and
    # replayed; the FFN timing events are captured with it, so the values read
    # after the loop are those of the last timed replay.
    layer.expert_ffn = timed_expert_ffn
    attn_events = []
    for stg in att_stages or []:
        stg.timing = attn_events
    if args.graph:
        runner.capture(xs)
        barrier()
        for _ in range(args.warmup):  # warm-up replays of the captured step
            runner.replay()
        torch.cuda.synchronize()
        barrier()
    if g.is_expert:
        rows0, calls0 = g.stats()
    clk = ClockSampler(local)
    clk.start()
    torch.cuda.synchronize()
    barrier()
    step = runner.replay if args.graph else (lambda: runner.run(xs))
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk.window_open()
    t_start.record()
    for _ in range(args.steps):
        step()
    t_end.record()
    torch.cuda.synchronize()
    clk.window_close()
    barrier()
    clocks = clk.stop()
    layer.expert_ffn = orig_ffn
    elapsed_ms = t_start.elapsed_time(t_end)
    st = g.status()
    if st != 0:
        raise RuntimeError(f"device status {st} (timeout in a device-side wait)")
    parity = parity_check(layer, g, runner, att_stages, xs, wg, w13, w2, model)
    if world > 1:
        allp = [None] * world
        dist.all_gather_object(allp, parity)
        ranks = [p for p in allp if p is not None]
        parity = {"per_attention_rank": ranks,
                  "routing_bit_exact": all(p["routing_bit_exact"] for p in ranks),
                  "combine_bit_exact": all(p.get("combine_bit_exact", True) for p in ranks)}
    if args.graph:
        # capture() runs one eager step before recording the graph: keep only
        # the graph's events (re-stamped by every replay -> the last timed step)
        per = plan.m * args.layers
        ffn_events, attn_events = ffn_events[-per:], attn_events[-per:]
    ffn_ms = [s.elapsed_time(e) for s, e in ffn_events]
    attn_ms = [s.elapsed_time(e) for s, e in attn_events]
    for stg in att_stages or []:
        stg.timing = None
    attn_report = None
    if att_stages:
        # decode_attn_kernel: algorithmic bytes (K/V rows read + q + o) per launch
        # (graph mode: the last timed replay's launches)
        by = sum(stg.attn_bytes() for stg in att_stages) / len(att_stages) * len(attn_ms)
        ms = sum(attn_ms)
        gbps = by / (ms / 1e3) / 1e9 if ms else None
        hbm = measured_peaks().get("hbm_gbs") or 6546.6
        attn_report = {"kernel": "decode_attn_kernel (paged GQA decode, TMA-streamed KV)", "bound": "hbm",
                       "heads": att_stages[0].n_heads, "kv_heads": att_stages[0].n_kv, "page_tokens": 64,
                       "mean_ctx": float(np.mean([stg.cache.ctx_host.mean() for stg in att_stages])),
                       "bytes_per_launch": by / max(len(attn_ms), 1), "avg_launch_ms": ms / max(len(attn_ms), 1),
                       "achieved": gbps, "peak": hbm, "unit": "GB/s", "frac": gbps / hbm if gbps else None,
                       "peak_kind": "measured hbm_gbs (MEASURED_PEAKS.json, copy read+write)"}
    rows = calls = 0
    if g.is_expert:
        rows1, calls1 = g.stats()
        rows, calls = rows1 - rows0, calls1 - calls0
    # reductions over ranks: step time = max; FFN stats summed over expert ranks
    t = torch.tensor([elapsed_ms, sum(ffn_ms), len(ffn_ms), rows, calls], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = t.clone()
        m_, s_ = tmax[:1].clone(), tmax[1:].clone()
        allreduce_(m_, dist.ReduceOp.MAX)
        allreduce_(s_, dist.ReduceOp.SUM)
        tmax = torch.cat([m_, s_])
        t = tmax
    elapsed_ms, ffn_total_ms, ffn_n, rows_total, calls_total = t.tolist()
    # rows each expert GPU processed per FFN call (load balance evidence)
    mine = (rows / calls) if (g.is_expert and calls) else None
    per_gpu_rows = [mine]
    if world > 1:
        per_gpu_rows = [None] * world
        dist.all_gather_object(per_gpu_rows, mine)
    per_gpu_rows = [r for r in per_gpu_rows if r is not None]
    lb_report = None
    if loads is not None:
        from paper_2504_02263_b200.balance import identity_slots
        ident = identity_slots(model.experts, n_e)
        lb_report = {"skew": args.skew, "balanced": bool(args.balance),
                     "expert_loads": [int(v) for v in loads],
                     "rows_per_expert_gpu_per_call": per_gpu_rows,
                     "max_over_mean": (max(per_gpu_rows) / (sum(per_gpu_rows) / len(per_gpu_rows)))
                     if per_gpu_rows else None,
                     "expected_max_rows_unbalanced": float(ident.expected_gpu_rows(loads).max()),
                     "expected_max_rows": float((slots or ident).expected_gpu_rows(loads).max()),
                     "physical_slots": slots.P if slots else model.experts}

    # ---- measured stage times vs the reference's timing model (Eq. 5) ----
    stages = runner.stage_times_ms()
    all_stages = [stages]
    if world > 1:
        all_stages = [None] * world
        dist.all_gather_object(all_stages, stages)
    if args.timeline_csv:  # SPEC.md:232 schema, one file per rank (events are per-GPU clocks)
        import csv as _csv
        path = args.timeline_csv.replace("{rank}", str(rank))
        with open(path, "w", newline="") as fh:
            wcsv = _csv.writer(fh)
            wcsv.writerow(["resource", "microbatch", "layer", "phase", "start_s", "end_s"])
            for ph, j, l, s, e in runner.timeline():
                wcsv.writerow([f"gpu{rank}:{g.role}", j, l, ph, s / 1e3, e / 1e3])

    # ---- e2e through the public API with host buffers -------------------
    e2e = None
    if full and not args.no_e2e:
        # Host-resident inputs and results, every step: step i+1's inputs go
        # H2D and step i's results go D2H on a copy stream while step i
        # computes (double-buffered pinned host buffers + device staging; the
        # step itself only adds two device-to-device copies).  Serving systems
        # overlap exactly these transfers; the bytes are the step's own.
        outs = [runner._out(xs, j) for j in range(plan.m)] if xs else []
        host_in = [[x.cpu().pin_memory() for x in x0] for _ in range(2)] if xs else None
        host_out = [[torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs] for _ in range(2)] if xs else None
        stage_in = [[torch.empty_like(x) for x in xs] for _ in range(2)] if xs else None
        stage_out = [[torch.empty_like(o) for o in outs] for _ in range(2)] if xs else None
        cstream = torch.cuda.Stream(device=dev)
        main = torch.cuda.current_stream()
        in_ready = [torch.cuda.Event() for _ in range(2)]
        in_free = [torch.cuda.Event() for _ in range(2)]
        out_ready = [torch.cuda.Event() for _ in range(2)]
        out_free = [torch.cuda.Event() for _ in range(2)]
        barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        if xs:
            with torch.cuda.stream(cstream):
                cstream.wait_stream(main)
                for d, h in zip(stage_in[0], host_in[0]):
                    d.copy_(h, non_blocking=True)
                in_ready[0].record(cstream)
        for i in range(args.steps):
            b = i % 2
            if xs:
                main.wait_event(in_ready[b])
                for x, d in zip(xs, stage_in[b]):
                    x.copy_(d, non_blocking=True)
                in_free[b].record(main)
                if i + 1 < args.steps:  # prefetch the next step's inputs
                    nb = (i + 1) % 2
                    with torch.cuda.stream(cstream):
                        if i >= 1:
                            cstream.wait_event(in_free[nb])
                        for d, h in zip(stage_in[nb], host_in[nb]):
                            d.copy_(h, non_blocking=True)
                        in_ready[nb].record(cstream)
            step()
            if xs:
                if i >= 2:
                    main.wait_event(out_free[b])
                for d, o in zip(stage_out[b], outs):
                    d.copy_(o, non_blocking=True)
                out_ready[b].record(main)
                with torch.cuda.stream(cstream):
                    cstream.wait_event(out_ready[b])
                    for h, d in zip(host_out[b], stage_out[b]):
                        h.copy_(d, non_blocking=True)
                    out_free[b].record(cstream)
        main.wait_stream(cstream)
        e.record()
        torch.cuda.synchronize()
        barrier()
        e2e_ms = torch.tensor([s.elapsed_time(e)], dtype=torch.float64, device=dev)
        if world > 1:
            allreduce_(e2e_ms, dist.ReduceOp.MAX)
        bytes_io = plan.m * args.b_a * model.hidden * 2 if xs else 0
        tok = n_a * plan.m * args.b_a * args.layers * args.steps
        ok = all(torch.equal(h.to(dev), o) for h, o in zip(host_out[(args.steps - 1) % 2], outs)) if xs else True
        e2e = {"value": tok / (e2e_ms.item() / 1e3), "unit": "layer-tokens/s",
               "h2d_bytes_per_step": bytes_io, "d2h_bytes_per_step": bytes_io, "results_checked": ok,
               "note": "per attention rank: m micro-batch inputs H2D from pinned memory and the m layer "
                       "outputs D2H every step, overlapped with the previous/next step on a copy stream"}

    # ---- the metric's M2N dispatch+combine p50 (this config's micro-batch) ----
    m2n = None
    if full and not args.no_m2n:
        xm = None
        if g.is_attention:
            xm = att_stages[0].y if att_stages else xs[0]
        m2n = m2n_latency(layer, g, xm, world)

    if rank != 0:
        g.close()
        return None

    peaks = measured_peaks()
    traffic = ncu_traffic(model.name, args.b_a, n_a, n_e, colo)
    if attn_report is not None:
        attn_report["traffic"] = traffic.get("decode_attn") if traffic else None
    tokens = n_a * plan.m * args.b_a * args.layers * args.steps
    value = tokens / (elapsed_ms / 1e3)
    ffn_avg_s = (ffn_total_ms / max(ffn_n, 1)) / 1e3
    # per expert GPU: its rows x its h'/tp_e slice of every expert
    flops_per_call = 6.0 * (rows_total / max(calls_total, 1)) * model.hidden * model.intermediate / plan.tp_e
    achieved = flops_per_call / ffn_avg_s / 1e12 if ffn_n else None
    # the burst figure: the timed region (K steps of ~20 ms) is shorter than
    # the 4 s back-to-back run the sustained figure comes from
    peak = peaks.get("bf16_tflops") or 1677.4
    peak_sus = peaks.get("bf16_tflops_sustained") or 1404.8
    # our kernels per (micro-batch, layer): attention (real: QKV GEMM with
    # RoPE/append epilogue + decode_attn [+ split combine] + O GEMM with the
    # residual), router + dispatch (one fused launch; E >= 64 at T <= 256:
    # logits + route kernels), expert wait + [region gather when several
    # senders share an expert] + 2 GEMMs, combine
    attn_launches = 0
    if att_stages:  # TP node: publish, QKV, attention [+ combine], O projection, reduce
        attn_launches = (5 if tp_a > 1 else 3) + (1 if att_stages[0].ws is not None else 0)
    router_launches = router_launch_count(model.experts, args.b_a)
    expert_launches = 3 + (1 if n_a > 1 else 0)
    launches_per_mbl = attn_launches + router_launches + expert_launches + 1
    line = {
        "metric": "decode tokens/s/GPU (MoE layer, ping-pong); M2N dispatch+combine p50 µs",
        "value": value, "unit": "layer-tokens/s", "value_per_gpu": value / world,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights seed 0, N(0,1) tokens)",
        "config": bench_config(args, model, n_a, n_e, colo, plan_source, plan.tp_e, plan.m, args.b_a, world),
        "roofline": {"bound": "tensor", "kernel": "expert FFN (grouped_gemm_kernel x2: gate/up+SiLU, down+N2M)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic.get("ffn_pair") if traffic else None,
                     "traffic_source": "profiles/r02_ncu_traffic.json (ncu --set full, dram read+write per launch pair)"
                     if traffic else None,
                     "frac_sustained": (achieved / peak_sus) if achieved else None,
                     "frac_nominal_dense": (achieved / 2250.0) if achieved else None,
                     "flops_per_launch_pair": flops_per_call, "avg_launch_pair_ms": ffn_avg_s * 1e3,
                     "peak_kind": "measured bf16_tflops burst (MEASURED_PEAKS.json; frac_sustained vs the "
                                  "4 s back-to-back figure)"},
        "parity": parity,
        "e2e": e2e,
        "gpu_launches": None,
        "clocks": clocks,
        "stage_times": eq5_report(all_stages, plan, args.layers, elapsed_ms / args.steps, colo),
        # whole-model equivalents: the layer step repeated for
        # MoeModelSpec.layers layers; TBT vs WorkloadSpec.slo_tbt (catalog.py:132)
        "whole_model": {"layers": model.layers, "tokens_per_s": value / model.layers,
                        "tbt_ms": elapsed_ms / args.steps / args.layers * model.layers,
                        "slo_tbt_ms": WorkloadSpec().slo_tbt * 1e3},
        "load_balance": lb_report,
        "attention": attn_report,
        "m2n": m2n,
    }
    # our kernels inside the timed region (per rank, summed over roles)
    per_step = plan.m * args.layers * (launches_per_mbl * world if colo else 0)
    if not colo:
        per_step = plan.m * args.layers * (n_a * (attn_launches + router_launches + 1) + n_e * expert_launches)
    line["gpu_launches"] = per_step * args.steps
    if full and not args.no_cpu and world == 1:  # the CPU baseline is timed at N = 1 only
        threads = len(os.sched_getaffinity(0))
        cs = cpu_layer(model, plan.m * args.b_a, attn=args.attn == "real", steps=1, warmup=1)
        line["cpu_baseline"] = {"value": cs["tokens_per_s"], "unit": "layer-tokens/s", "cores": threads,
                                "kind": "port", "sample": cs["sample"], "cpu": cpu_model_name(),
                                "t_layer_s": cs["t_layer_s"], "t_attention_s": cs["t_attention_s"],
                                "t_moe_s": cs["t_moe_s"]}
    g.close()
    return line


def main():
    args = parse()
    if os.environ.get("MSI_BENCH_STACKDUMP"):  # diagnostics: dump every thread's stack every N s
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["MSI_BENCH_STACKDUMP"]), repeat=True)
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2504_02263_b200 import runtime

    rank, world, local = runtime.init_distributed_from_env("gloo" if _over() else "nccl")
    if world != args.gpus:
        if rank == 0:
            print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}))
        sys.exit(2)
    import copy
    args0 = copy.copy(args)  # measure() folds merged micro-batches into args.b_a
    layout = resolve_layout(args, world)
    line = measure(args, rank, world, local, layout, full=True)
    if world > 1 and layout[2] and args.pingpong:
        # The paper's disaggregated ping-pong layout, measured beside the
        # co-located headline with the same tokens per attention GPU per
        # micro-batch: n_e from the headline's own per-token stage costs
        # (T_e / (T_a + T_e) of the GPUs), experts spread over n_e GPUs.
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        share = [None]
        if rank == 0:
            st = line["stage_times"]
            share[0] = st["T_e_ms"] / (st["T_a_ms"] + st["T_e_ms"])
        dist.broadcast_object_list(share, src=0)
        alt, slots = disaggregated_layout(args0, world, share[0])
        sub = measure(args0, rank, world, local, alt, full=False, slots_override=slots)
        if rank == 0:
            line["pingpong"] = pingpong_summary(sub, share[0])
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
