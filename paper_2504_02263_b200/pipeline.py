"""Ping-pong micro-batch pipeline: the reference's timing model of the path.

The reference specifies (not shipped) closed forms and a
discrete-event simulator of m micro-batches x L layers over two exclusive
resources (attention group, expert group) joined by a delay link.  This module
restates them so the measured B200 pipeline (``runtime.MoEDecodeLayer``) can be
checked against Eq. 5 and emit the same timeline schema
(resource, microbatch, layer, phase in {attn, disp, ffn, comb}, start, end),
SPEC.md:232 / 298.
"""

from __future__ import annotations

import csv
import heapq
import math
from dataclasses import dataclass, field

PHASES = ("attn", "disp", "ffn", "comb")


@dataclass(frozen=True)
class StageTimes:
    """T_a, T_e, T_c in seconds; T_f = max(T_a, T_e)."""

    T_a: float
    T_e: float
    T_c: float

    def __post_init__(self):
        if min(self.T_a, self.T_e, self.T_c) < 0:
            raise ValueError("stage times must be >= 0")

    @property
    def T_f(self) -> float:
        return max(self.T_a, self.T_e)


def min_microbatches(T_c: float, T_f: float) -> int:
    """Smallest m with m >= 2(1 + T_c/T_f).

    Raises ValueError when T_c >= T_f (constraint 2: communication cannot be
    hidden behind compute)."""
    if T_f <= 0 or T_c < 0:
        raise ValueError("need T_f > 0 and T_c >= 0")
    if T_c >= T_f:
        raise ValueError("communication not hideable: T_c >= T_f (constraint 2)")
    need = 2.0 * (1.0 + T_c / T_f)
    # tolerate 2(1 + x) landing a hair above an integer through rounding
    return max(2, math.ceil(need - 1e-12))


def closed_form_total(t: StageTimes, m: int, L: int) -> float:
    """Eq. 5: T_total = (T_a + T_e + 2 T_c) + T_f (m L - 1)."""
    if m < 1 or L < 1:
        raise ValueError("m and L must be >= 1")
    return (t.T_a + t.T_e + 2 * t.T_c) + t.T_f * (m * L - 1)


def closed_form_iter_bounds(t: StageTimes, m: int, L: int) -> tuple[float, float]:
    """Eq. 4: (T_a+T_e+2T_c) + m T_f (L-1) <= T_iter <= m T_f L."""
    if m < 1 or L < 1:
        raise ValueError("m and L must be >= 1")
    lower = (t.T_a + t.T_e + 2 * t.T_c) + m * t.T_f * (L - 1)
    return lower, m * t.T_f * L


@dataclass
class SimReport:
    iter_latency_per_microbatch: float
    total_latency: float
    attention_idle_fraction: float
    expert_idle_fraction: float
    timeline: list = field(default_factory=list)

    def write_timeline_csv(self, path) -> None:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["resource", "microbatch", "layer", "phase", "start_s", "end_s"])
            w.writerows(self.timeline)


def simulate(t: StageTimes, m: int, L: int) -> SimReport:
    """Deterministic event simulation of the ping-pong schedule.

    Two exclusive resources process ready work FIFO (earliest-ready first,
    then micro-batch index); dispatch/combine are pure delays of T_c on a
    non-blocking link.  Returns the timeline and the summary fields."""
    if m < 1 or L < 1:
        raise ValueError("m and L must be >= 1")
    dur = {"attention": t.T_a, "expert": t.T_e}
    free_at = {"attention": 0.0, "expert": 0.0}
    busy = {"attention": 0.0, "expert": 0.0}
    # pending: (ready, mb, layer, resource)
    pending: list[tuple[float, int, int, str]] = [(0.0, j, 0, "attention") for j in range(m)]
    heapq.heapify(pending)
    timeline = []
    first_start = {}
    last_end = {}
    while pending:
        # pick the task with the earliest feasible start, FIFO on ties
        best = min(pending, key=lambda p: (max(p[0], free_at[p[3]]), p[0], p[1]))
        pending.remove(best)
        ready, j, layer, res = best
        start = max(ready, free_at[res])
        end = start + dur[res]
        free_at[res] = end
        busy[res] += dur[res]
        if res == "attention":
            timeline.append((res, j, layer, "attn", start, end))
            first_start.setdefault(j, start)
            timeline.append(("link", j, layer, "disp", end, end + t.T_c))
            pending.append((end + t.T_c, j, layer, "expert"))
        else:
            timeline.append((res, j, layer, "ffn", start, end))
            timeline.append(("link", j, layer, "comb", end, end + t.T_c))
            if layer + 1 < L:
                pending.append((end + t.T_c, j, layer + 1, "attention"))
            else:
                last_end[j] = end + t.T_c
    total = max(last_end.values())
    per_mb = sum(last_end[j] - first_start[j] for j in range(m)) / m
    timeline.sort(key=lambda r: (r[4], r[0], r[1]))
    return SimReport(
        iter_latency_per_microbatch=per_mb,
        total_latency=total,
        attention_idle_fraction=1.0 - busy["attention"] / total if total else 0.0,
        expert_idle_fraction=1.0 - busy["expert"] / total if total else 0.0,
        timeline=timeline,
    )
