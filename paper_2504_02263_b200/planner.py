"""Deployment-plan search (Algorithm 1) driven by B200-calibrated cost models
(SURVEY.md §8(f) rank 4).

Two searches share the same evaluation:

* ``search``      -- Algorithm 1 as printed:
  tp_e, tp_a over {1, 2, 4, 8} (<= max_gpus_per_node), memory check
  (tp_a C_a > P_a and tp_e C_e > P_e), n_a from ``balance_attention_nodes``,
  m in {3 .. N_m}, the largest global batch B under the SLO by binary search,
  argmax of throughput per unit cost (tpuc) with the SPEC's tie-break (fewer
  GPUs, then smaller m, then smaller tp_a).  One expert per expert node.
* ``search_box``  -- the same objective on one 8xB200 NVSwitch box as this
  runtime deploys it: n_a attention GPUs + n_e expert nodes of tp_e GPUs
  (E_l = E / n_e experts each, h' split tp_e ways), or all GPUs co-located,
  m micro-batches, per-GPU b_a.  This is what chooses ``bench.py``'s layout
  from measured coefficients.

Per candidate: b_e = B K / (m E_nodes) rows per expert
node per micro-batch, T_a = k1 b_a + k2, T_e = k3 b_e + k4, T_c = Eq. 6,
T_f = max(T_a, T_e); feasible iff |T_a - T_e| / T_f <= balance_slack
(constraint 1), T_c < T_f (2), m >= min_microbatches (3), the KV + attention
parameter memory 4 m b_a s h L / g + P_a < tp_a C_a (7), and the SLO on the
Eq. 4 upper bound T_iter = m T_f L.  tpuc = (B / T_total) / (cost of all
GPUs) with T_total from Eq. 5.
"""

from __future__ import annotations

import math
from dataclasses import asdict, dataclass, field

from . import perf_model as PM
from .config import ConfigError, GpuSpec, MoeModelSpec, SearchLimits, WorkloadSpec
from .pipeline import StageTimes, closed_form_total, min_microbatches

TP_CHOICES = (1, 2, 4, 8)


# ---------------------------------------------------------------- sizing ----
def param_sizes(model: MoeModelSpec, swiglu: bool = False) -> tuple[int, int]:
    """(P_a, P_e) bytes over all layers: P_a = L h^2 (2 + 2/g) bytes,
    P_e = L 2 h h' bytes per expert (3 h h' with ``swiglu``, what the runtime executes)."""
    b = model.bytes_per_param
    p_a = model.layers * model.hidden * model.hidden * (2 + 2 / model.gqa_group) * b
    p_e = model.layers * (3 if swiglu else 2) * model.hidden * model.intermediate * b
    return int(p_a), int(p_e)


def kv_bytes(m: int, b_a: float, model: MoeModelSpec, seq_len: float) -> float:
    """Constraint 7's KV term 4 m b_a s h L / g."""
    return 4.0 * m * b_a * seq_len * model.hidden * model.layers / model.gqa_group


def balance_attention_nodes(cm: PM.CostModel, E: int, K: int, b_ref: float = 1.0) -> int:
    """n_a = (k1 E) / (k3 K) rounded to the neighbour that minimises |T_a - T_e|
    at the representative batch b_ref (tie -> smaller), clamped >= 1
    (SPEC.md:311-318)."""
    x = cm.k1 * E / (cm.k3 * K)
    cands = sorted({max(1, math.floor(x)), max(1, math.ceil(x))})

    def gap(n):
        b_e = b_ref * n * K / E
        return abs(PM.attention_time(b_ref, cm) - PM.expert_time(b_e, cm))

    return min(cands, key=lambda n: (gap(n), n))


# ------------------------------------------------------------- candidates ----
@dataclass
class Plan:
    tp_a: int
    tp_e: int
    n_a: int
    n_e: int           # expert nodes (paper: E nodes of tp_e GPUs; box: expert GPUs)
    m: int
    B: int             # global batch (tokens per decode iteration)
    b_a: float
    b_e: float
    T_a: float
    T_e: float
    T_c: float
    T_f: float
    T_iter_upper: float
    T_total: float
    tpuc: float
    gpus: int
    colocated: bool = False
    slack: dict = field(default_factory=dict)

    def to_dict(self) -> dict:
        return asdict(self)


@dataclass
class NoPlan:
    """Empty search: the binding constraint per rejected candidate."""

    reasons: list

    def __bool__(self):
        return False


def _tp_scaled(cm: PM.CostModel, tp_a: int, tp_e: int) -> PM.CostModel:
    """Per-tp coefficients: slopes divide by tp (ideal TP split of the per-token
    work), intercepts stay (fixed costs per GPU)."""
    return PM.CostModel(k1=cm.k1 / tp_a, k2=cm.k2, k3=cm.k3 / tp_e, k4=cm.k4, util_curve=cm.util_curve,
                        comm_backend=cm.comm_backend)


def evaluate(model: MoeModelSpec, gpu_a: GpuSpec, gpu_e: GpuSpec, cm: PM.CostModel, workload: WorkloadSpec,
             tp_a: int, tp_e: int, n_a: int, n_e: int, m: int, B: int, balance_slack: float = 0.10,
             colocated: bool = False, swiglu: bool = False, expert_nodes_hold: int = 1,
             cost_metric: str = "price") -> tuple[Plan | None, str]:
    """Evaluate one candidate at global batch B -> (Plan, "") or (None, binding constraint)."""
    L, K = model.layers, model.topk
    b_a = B / (m * n_a)
    b_e = B * K / (m * n_e)
    t_a = PM.attention_time(b_a, cm, None)
    t_e = PM.expert_time(b_e, cm)
    if colocated:
        # both roles on every GPU, M2N stays inside the box; no ping-pong partner
        t_c = 0.0
        t_f = t_a + t_e
        t_total = m * L * t_f
        t_iter = t_total
    else:
        t_c = PM.comm_time(b_a, b_e, model.hidden, K, tp_a, tp_e, gpu_a.net_bandwidth_per_gpu * tp_a,
                           gpu_e.net_bandwidth_per_gpu * tp_e, cm, model.bytes_per_param)
        t_f = max(t_a, t_e)
        if abs(t_a - t_e) / t_f > balance_slack:
            return None, "balance (constraint 1)"
        if not t_c < t_f:
            return None, "communication not hidden (constraint 2: T_c < T_f)"
        if m < min_microbatches(t_c, t_f):
            return None, "too few micro-batches (constraint 3)"
        t_total = closed_form_total(StageTimes(t_a, t_e, t_c), m, L)
        t_iter = m * t_f * L
    if t_iter > workload.slo_tbt:
        return None, "SLO"
    p_a, p_e = param_sizes(model, swiglu)
    if kv_bytes(m, b_a, model, workload.avg_seq_len) + p_a >= tp_a * gpu_a.mem_capacity:
        return None, "attention memory (constraint 7)"
    if expert_nodes_hold * p_e >= tp_e * gpu_e.mem_capacity:
        return None, "expert memory"
    gpus = n_a * tp_a + (0 if colocated else n_e * tp_e)
    unit_a = gpu_a.price if cost_metric == "price" else (gpu_a.max_power or float("nan"))
    unit_e = gpu_e.price if cost_metric == "price" else (gpu_e.max_power or float("nan"))
    cost = n_a * tp_a * unit_a + (0 if colocated else n_e * tp_e * unit_e)
    tpuc = (B / t_total) / cost
    slack = {"balance": abs(t_a - t_e) / t_f, "comm_over_Tf": t_c / t_f if t_f else 0.0,
             "slo": workload.slo_tbt - t_iter,
             "attn_mem_bytes": tp_a * gpu_a.mem_capacity - kv_bytes(m, b_a, model, workload.avg_seq_len) - p_a}
    return Plan(tp_a, tp_e, n_a, n_e, m, int(B), b_a, b_e, t_a, t_e, t_c, t_f, t_iter, t_total, tpuc, gpus,
                colocated, slack), ""


def max_batch_under_slo(model, gpu_a, gpu_e, cm, workload, tp_a, tp_e, n_a, n_e, m, b_max: int = 1 << 22,
                        **kw) -> tuple[Plan | None, str]:
    """Largest B (multiple of m n_a) whose plan is feasible.
    Feasibility is monotone in B above the balance region for the SLO and
    memory constraints; the binary search runs on the upper constraints and
    the result is re-checked with every constraint."""
    step = m * n_a
    lo, hi = 0, b_max // step  # feasible in units of step: search the largest k with B = k*step
    reason = "SLO"

    kw_upper = dict(kw, balance_slack=float("inf"))

    def upper_ok(k):
        p, r = evaluate(model, gpu_a, gpu_e, cm, workload, tp_a, tp_e, n_a, n_e, m, k * step, **kw_upper)
        return p is not None, r

    ok, r = upper_ok(1)
    if not ok and r in ("SLO", "attention memory (constraint 7)", "expert memory"):
        return None, r
    while lo < hi:
        mid = (lo + hi + 1) // 2
        ok, r = upper_ok(mid)
        if ok or r not in ("SLO", "attention memory (constraint 7)", "expert memory"):
            lo = mid
        else:
            hi, reason = mid - 1, r
    if lo == 0:
        return None, reason
    return evaluate(model, gpu_a, gpu_e, cm, workload, tp_a, tp_e, n_a, n_e, m, lo * step, **kw)


def _better(p: Plan, best: Plan | None) -> bool:
    if best is None:
        return True
    if p.tpuc != best.tpuc:
        return p.tpuc > best.tpuc
    return (p.gpus, p.m, p.tp_a) < (best.gpus, best.m, best.tp_a)


def search(model: MoeModelSpec, gpu_a: GpuSpec, gpu_e: GpuSpec, cm: PM.CostModel, workload: WorkloadSpec,
           limits: SearchLimits = SearchLimits(), balance_slack: float = 0.10, swiglu: bool = False,
           explain: list | None = None) -> Plan | NoPlan:
    """Algorithm 1."""
    p_a, p_e = param_sizes(model, swiglu)
    best, reasons = None, []
    for tp_e in [t for t in TP_CHOICES if t <= gpu_e.max_gpus_per_node]:
        for tp_a in [t for t in TP_CHOICES if t <= gpu_a.max_gpus_per_node]:
            if not (tp_a * gpu_a.mem_capacity > p_a and tp_e * gpu_e.mem_capacity > p_e):
                reasons.append(((tp_a, tp_e), "parameter memory (Alg. 1 line 4)"))
                continue
            cmt = _tp_scaled(cm, tp_a, tp_e)
            n_a = balance_attention_nodes(cmt, model.experts, model.topk)
            for m in range(3, limits.max_microbatches + 1):
                p, r = max_batch_under_slo(model, gpu_a, gpu_e, cmt, workload, tp_a, tp_e, n_a, model.experts, m,
                                           balance_slack=balance_slack, swiglu=swiglu,
                                           cost_metric=limits.cost_metric)
                if explain is not None:
                    explain.append({"tp_a": tp_a, "tp_e": tp_e, "n_a": n_a, "m": m,
                                    "tpuc": p.tpuc if p else None, "B": p.B if p else None, "reason": r})
                if p is None:
                    reasons.append(((tp_a, tp_e, m), r))
                elif _better(p, best):
                    best = p
    return best if best is not None else NoPlan(reasons)


def _head_layout(model) -> tuple[int, int]:
    """(n_heads, n_kv) as the attention stage lays them out (attention.head_layout)."""
    n_heads = max(1, model.hidden // 128)
    g = max(1, min(int(getattr(model, "gqa_group", 8)), n_heads, 16))
    while n_heads % g:
        g -= 1
    return n_heads, n_heads // g


def search_box(model: MoeModelSpec, gpu: GpuSpec, cm_for, workload: WorkloadSpec, n_gpus: int = 8,
               max_microbatches: int = 4, balance_slack: float = 0.25, swiglu: bool = True,
               explain: list | None = None, tp_choices=(1, 2, 4), tp_a_choices=(1, 2, 4)) -> Plan | NoPlan:
    """One B200 box: n_a attention GPUs + n_e expert nodes of tp_e GPUs
    (n_a + n_e tp_e = n_gpus, E divisible by n_e) with m in {2..N_m}, or all
    GPUs co-located (m = 1, merged batch).  ``cm_for(E_l)`` returns the cost
    model calibrated for E_l local experts per expert GPU (the expert
    intercept is the weight stream of those E_l experts); with expert TP each
    GPU streams E_l / tp_e experts' weights and does 1 / tp_e of the per-row
    work.  The returned Plan's n_e counts expert nodes (GPUs = n_e tp_e) and
    its n_a attention nodes of tp_a GPUs (heads split; the attention slope
    k1 divides by tp_a -- the all-gather / reduce-scatter ride on NVLink
    inside the projection GEMMs, attn_tp.cu)."""
    best, reasons = None, []
    E = model.experts
    _, n_kv = _head_layout(model)
    cands = [((n_gpus - nodes * tp) // tpa, nodes, tp, tpa, False)
             for tp in tp_choices for tpa in tp_a_choices for nodes in range(1, n_gpus)
             if 0 < nodes * tp < n_gpus and (n_gpus - nodes * tp) % tpa == 0 and n_kv % tpa == 0
             and E % nodes == 0 and model.intermediate % (128 * tp) == 0]
    if E % n_gpus == 0:
        cands.append((n_gpus, n_gpus, 1, 1, True))
    for n_a, n_e, tp, tpa, colo in cands:
        E_l = E // n_e
        cm = cm_for(E_l / tp)
        cm = PM.CostModel(k1=cm.k1 / tpa, k2=cm.k2, k3=cm.k3 / tp, k4=cm.k4, util_curve=cm.util_curve,
                          comm_backend=cm.comm_backend)
        for m in ([1] if colo else range(2, max_microbatches + 1)):
            p, r = max_batch_under_slo(model, gpu, gpu, cm, workload, tpa, tp, n_a, n_e, m,
                                       balance_slack=balance_slack, colocated=colo, swiglu=swiglu,
                                       expert_nodes_hold=E_l)
            if explain is not None:
                explain.append({"n_a": n_a, "tp_a": tpa, "n_e": n_e, "tp_e": tp, "colocated": colo, "m": m,
                                "tpuc": p.tpuc if p else None, "B": p.B if p else None, "reason": r})
            if p is None:
                reasons.append(((n_a, tpa, n_e, tp, m), r))
            elif _better(p, best):
                best = p
    return best if best is not None else NoPlan(reasons)


def cm_scaled_for_experts(cm: PM.CostModel, e_l_calibrated: int):
    """``cm_for`` from one calibration at e_l_calibrated local experts: the
    expert intercept k4 (weight streaming) scales with E_l."""
    if e_l_calibrated < 1:
        raise ConfigError("e_l_calibrated must be >= 1")

    def f(E_l: int) -> PM.CostModel:
        return PM.CostModel(k1=cm.k1, k2=cm.k2, k3=cm.k3, k4=cm.k4 * E_l / e_l_calibrated,
                            util_curve=cm.util_curve, comm_backend=cm.comm_backend)

    return f


def to_deployment(p: Plan, b_a: int | None = None):
    """A ``search_box`` result as the runtime's ``config.DeploymentPlan``
    (expert GPUs = nodes x tp_e; b_a defaults to the plan's per-GPU batch)."""
    from .config import DeploymentPlan

    if not p:
        raise ConfigError("to_deployment: empty search result")
    ba = int(b_a if b_a is not None else max(1, round(p.b_a)))
    if p.colocated:
        return DeploymentPlan(n_a=p.n_a, n_e=p.n_a, m=p.m, b_a=ba, colocated=True)
    if b_a is None:  # the plan's b_a is per attention node: each of its tp_a GPUs holds a shard
        ba = max(1, round(p.b_a / p.tp_a))
    return DeploymentPlan(n_a=p.n_a * p.tp_a, n_e=p.n_e * p.tp_e, m=p.m, b_a=ba, tp_e=p.tp_e, tp_a=p.tp_a)


def main(argv=None) -> int:
    """Plan JSON output: run Algorithm 1 on one B200 box with calibrated
    coefficients and write the config + ``plan`` section that ``load_plan`` /
    ``bench.py --plan-json`` read.

      python -m paper_2504_02263_b200.planner --model mixtral-8x22b \
          --calibration profiles/r01_calibration_8x22b.json --gpus 8 --out plan.json
    """
    import argparse
    import json

    from .config import Catalog, ConfigBundle, SearchLimits, as_model_spec, b200_gpu, load_config, save_plan

    ap = argparse.ArgumentParser(description=main.__doc__)
    ap.add_argument("--config", help="config JSON (model/workload/limits); default: builtin model")
    ap.add_argument("--model", default="mixtral-8x22b")
    ap.add_argument("--calibration", required=True, help="calibrate.py JSON (k1..k4, util table)")
    ap.add_argument("--gpus", type=int, default=8)
    ap.add_argument("--b-a", dest="b_a", type=int, default=None, help="per-GPU micro-batch (default: the plan's)")
    ap.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    if a.config:
        bundle = load_config(a.config)
    else:
        gpu = b200_gpu()
        bundle = ConfigBundle(Catalog([gpu]), as_model_spec(a.model), WorkloadSpec(), SearchLimits())
    with open(a.calibration) as fh:
        c = json.load(fh)
    cm = PM.CostModel(k1=c["k1_s_per_tok"], k2=c["k2_s"], k3=c["k3_s_per_tok"], k4=c["k4_s"],
                      util_curve=PM.UtilCurve.from_points(c["util_table"]))
    p = search_box(bundle.model, b200_gpu(), cm_scaled_for_experts(cm, c["experts_local"]), bundle.workload,
                   a.gpus)
    if not p:
        print(json.dumps({"error": "no feasible plan", "reasons": [list(map(str, r)) for r in p.reasons][:20]}))
        return 1
    dp = to_deployment(p, a.b_a)
    save_plan(bundle, dp, a.out, extra=p.to_dict())
    print(json.dumps({"plan": dp.__dict__, "tpuc": p.tpuc, "T_iter_upper": p.T_iter_upper, "out": a.out}))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
