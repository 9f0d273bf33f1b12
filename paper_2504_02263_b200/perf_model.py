"""Cost models of the MoE decode step, calibrated from B200 measurements
(SURVEY.md §8(f) rank 1).

The reference specifies these models but ships no code for them
(module ``perf_model``); this module restates the parts the
decode step's timing closes the loop with, under the same names:

* ``gemm_flops``                 SPEC.md:121-128 (2·b·h_in·h_out)
* ``min_compute_bound_batch``    SPEC.md:129-136 (ceil(F / BW))
* ``ffn_utilization``
* ``UtilCurve``                  SPEC.md:106-109 (parametric s_half or table)
* ``CommBackend``
* ``CostModel``                  SPEC.md:102-105 (k1..k4, alpha/beta)
* ``attention_time`` / ``expert_time``  SPEC.md:156-164 (affine)
* ``comm_time``                  SPEC.md:165-173 (Eq. 6)
* ``calibrate``                  SPEC.md:183-190 (least-squares affine fit)
* ``synthetic_points``           SPEC.md:186 (roofline oracle when no profile)
* ``read_profile`` / ``write_profile``  SPEC.md:211 (CSV ``kind,batch,seconds``
  and ``kind,message_bytes,utilization``)

On B200 the profile points come from ``calibrate.py`` (expert grouped GEMM
and attention stand-in timed with CUDA events, M2N utilisation from
``bench_m2n.py``); the fitted coefficients feed ``pipeline.StageTimes`` and
the Eq. 5 check in ``bench.py``.
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass, field
from typing import Iterable, Sequence

from .config import ConfigError

_INT64_MAX = (1 << 63) - 1


def gemm_flops(b: int, h_in: int, h_out: int) -> int:
    """2·b·h_in·h_out; errors on non-positive or overflow."""
    for v in (b, h_in, h_out):
        if not isinstance(v, int) or v <= 0:
            raise ConfigError("gemm_flops: arguments must be positive integers")
    f = 2 * b * h_in * h_out
    if f > _INT64_MAX:
        raise ConfigError("gemm_flops: overflow")
    return f


def min_compute_bound_batch(flops_per_s: float, bytes_per_s: float) -> int:
    """ceil(F / BW) tokens (312e12 / 2e12 -> 156)."""
    if not (flops_per_s > 0 and bytes_per_s > 0):
        raise ConfigError("min_compute_bound_batch: F and BW must be > 0")
    r = flops_per_s / bytes_per_s
    n = math.ceil(r)
    # guard float noise so an exact integer ratio is not bumped by one
    return n - 1 if n > 1 and abs((n - 1) - r) <= 1e-9 * r else n


def ffn_utilization(b: float, flops_per_s: float, bytes_per_s: float, moe: tuple | None = None) -> float:
    """min((K/E)·b·BW/F, 1) for MoE, min(b·BW/F, 1) dense."""
    if b < 0:
        raise ConfigError("ffn_utilization: b must be >= 0")
    u = b * bytes_per_s / flops_per_s
    if moe is not None:
        k, e = moe
        u *= k / e
    return min(max(u, 0.0), 1.0)


@dataclass(frozen=True)
class UtilCurve:
    """Bandwidth utilisation vs message size: parametric
    Util(x) = x/(x + s_half) (default s_half = 64 KiB) or a
    piecewise-linear table of (message_bytes, utilization), clamped at the ends."""

    s_half: float = 65536.0
    table: tuple = ()

    def __post_init__(self):
        if self.table:
            xs = [float(p[0]) for p in self.table]
            us = [float(p[1]) for p in self.table]
            if any(b <= a for a, b in zip(xs, xs[1:])):
                raise ConfigError("UtilCurve: table sizes must be strictly increasing")
            if any(not (0 < u <= 1) for u in us):
                raise ConfigError("UtilCurve: utilization must be in (0, 1]")
            if any(b < a for a, b in zip(us, us[1:])):
                raise ConfigError("UtilCurve: utilization must be non-decreasing")
        elif not self.s_half > 0:
            raise ConfigError("UtilCurve: s_half must be > 0")

    @classmethod
    def from_points(cls, points: Iterable[tuple]) -> "UtilCurve":
        """Table from measured points; enforces monotonicity by a running max
        (a measured dip at a larger size is noise, not capability)."""
        pts = sorted((float(x), float(u)) for x, u in points)
        out, best = [], 0.0
        for x, u in pts:
            best = max(best, min(u, 1.0))
            if out and out[-1][0] == x:
                out[-1] = (x, best)
            else:
                out.append((x, best))
        return cls(table=tuple(out))

    def __call__(self, x: float) -> float:
        if x <= 0:
            return self.table[0][1] if self.table else 0.0
        if not self.table:
            return x / (x + self.s_half)
        t = self.table
        if x <= t[0][0]:
            return t[0][1]
        if x >= t[-1][0]:
            return t[-1][1]
        for (x0, u0), (x1, u1) in zip(t, t[1:]):
            if x0 <= x <= x1:
                return u0 + (u1 - u0) * (x - x0) / (x1 - x0)
        return t[-1][1]


@dataclass(frozen=True)
class CommBackend:
    """Per-message cost parameters."""

    name: str = "nvlink-peer"
    base_overhead: float = 0.0
    per_receiver_penalty: float = 0.0
    jitter_p99_factor: float = 1.0

    def __post_init__(self):
        if self.base_overhead < 0 or self.per_receiver_penalty < 0:
            raise ConfigError("CommBackend: overheads must be >= 0")
        if self.jitter_p99_factor < 1:
            raise ConfigError("CommBackend: jitter_p99_factor must be >= 1")


@dataclass(frozen=True)
class CostModel:
    """k1..k4 with k1 = alpha·s + beta."""

    k1: float
    k2: float
    k3: float
    k4: float
    alpha: float = 0.0
    beta: float | None = None
    util_curve: UtilCurve = field(default_factory=UtilCurve)
    comm_backend: CommBackend = field(default_factory=CommBackend)

    def __post_init__(self):
        if not (self.k1 > 0 and self.k3 > 0):
            raise ConfigError("CostModel: k1 and k3 must be > 0")
        if self.k2 < 0 or self.k4 < 0 or self.alpha < 0:
            raise ConfigError("CostModel: k2, k4, alpha must be >= 0")

    def k1_at(self, s: float | None) -> float:
        if s is None or self.beta is None:
            return self.k1
        return self.alpha * s + self.beta


def attention_time(b_a: float, cm: CostModel, s: float | None = None) -> float:
    """T_a = k1·b_a + k2, k1 = alpha·s + beta when s is given."""
    if b_a < 0:
        raise ConfigError("attention_time: b_a must be >= 0")
    return cm.k1_at(s) * b_a + cm.k2


def expert_time(b_e: float, cm: CostModel) -> float:
    """T_e = k3·b_e + k4."""
    if b_e < 0:
        raise ConfigError("expert_time: b_e must be >= 0")
    return cm.k3 * b_e + cm.k4


def comm_time(b_a: float, b_e: float, hidden: int, topk: int, tp_a: int, tp_e: int,
              w_a: float, w_e: float, cm: CostModel, bytes_per_param: int = 2) -> float:
    """Eq. 6: max of the attention-side and expert-side
    directional times, each Util-derated at its message volume plus the
    backend's base overhead."""
    if min(b_a, b_e) < 0 or min(tp_a, tp_e) <= 0 or not (w_a > 0 and w_e > 0):
        raise ConfigError("comm_time: invalid arguments")
    va = b_a * hidden * topk * bytes_per_param / tp_a
    ve = b_e * hidden * bytes_per_param / tp_e
    ta = (va / (w_a * cm.util_curve(va)) if va > 0 else 0.0) + cm.comm_backend.base_overhead
    te = (ve / (w_e * cm.util_curve(ve)) if ve > 0 else 0.0) + cm.comm_backend.base_overhead
    return max(ta, te)


@dataclass(frozen=True)
class AffineFit:
    slope: float
    intercept: float
    residual_rms: float
    n: int

    def __call__(self, b: float) -> float:
        return self.slope * b + self.intercept


def calibrate(points: Sequence[tuple], kind: str = "expert") -> AffineFit:
    """Least-squares affine fit T(b) = slope·b + intercept.
    Errors on fewer than two distinct batch sizes.  The intercept is clamped
    at 0 (CostModel requires k2, k4 >= 0) and the slope refit through the
    origin when that happens."""
    if kind not in ("attention", "expert"):
        raise ConfigError("calibrate: kind must be 'attention' or 'expert'")
    pts = [(float(b), float(t)) for b, t in points]
    if len({b for b, _ in pts}) < 2:
        raise ConfigError("calibrate: need at least two distinct batch sizes")
    n = len(pts)
    mb = sum(b for b, _ in pts) / n
    mt = sum(t for _, t in pts) / n
    sbb = sum((b - mb) ** 2 for b, _ in pts)
    sbt = sum((b - mb) * (t - mt) for b, t in pts)
    slope = sbt / sbb
    icpt = mt - slope * mb
    if icpt < 0:
        icpt = 0.0
        slope = sum(b * t for b, t in pts) / sum(b * b for b, _ in pts)
    res = math.sqrt(sum((slope * b + icpt - t) ** 2 for b, t in pts) / n)
    return AffineFit(slope, icpt, res, n)


def synthetic_points(kind: str, batches: Sequence[int], hidden: int, inter: int,
                     flops_per_s: float, bytes_per_s: float, c0: float = 0.0,
                     seq_len: int = 730, gqa_group: int = 8, experts_local: int = 1,
                     bytes_per_param: int = 2) -> list:
    """Roofline oracle T(b) = max(flops(b)/F, bytes(b)/BW) + c0.
    expert: 2 Table-3 GEMMs (h->h', h'->h) over ``experts_local`` experts'
    weights; attention: QKV/output projections plus KV traffic 2·b·s·h·bytes/g."""
    out = []
    for b in batches:
        if kind == "expert":
            fl = 2 * 2.0 * b * hidden * inter
            by = experts_local * 2.0 * hidden * inter * bytes_per_param + 2.0 * b * hidden * bytes_per_param
        elif kind == "attention":
            g = gqa_group
            fl = 2.0 * b * hidden * hidden * (2 + 2 / g)
            by = hidden * hidden * (2 + 2 / g) * bytes_per_param + 2.0 * b * seq_len * hidden * bytes_per_param / g
        else:
            raise ConfigError("synthetic_points: kind must be 'attention' or 'expert'")
        out.append((b, max(fl / flops_per_s, by / bytes_per_s) + c0))
    return out


def write_profile(path: str, batch_rows: Iterable[tuple] = (), util_rows: Iterable[tuple] = ()) -> None:
    """CSV in the two SPEC.md:211 shapes: ``kind,batch,seconds`` rows, then
    ``kind,message_bytes,utilization`` rows (kind = backend name)."""
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kind", "batch", "seconds"])
        for r in batch_rows:
            w.writerow([r[0], int(r[1]), repr(float(r[2]))])
        util_rows = list(util_rows)
        if util_rows:
            w.writerow(["kind", "message_bytes", "utilization"])
            for r in util_rows:
                w.writerow([r[0], int(r[1]), repr(float(r[2]))])


def read_profile(path: str) -> tuple:
    """-> ({kind: [(batch, seconds)]}, {kind: [(message_bytes, utilization)]})."""
    batch, util = {}, {}
    mode = None
    with open(path, newline="") as f:
        for row in csv.reader(f):
            if not row or row[0].startswith("#"):
                continue
            if row[0] == "kind":
                mode = row[1]
                continue
            if mode == "batch":
                batch.setdefault(row[0], []).append((int(row[1]), float(row[2])))
            elif mode == "message_bytes":
                util.setdefault(row[0], []).append((int(row[1]), float(row[2])))
            else:
                raise ConfigError(f"{path}: row before a header")
    return batch, util


def cost_model_from_profile(path: str, seq_len: float | None = None) -> CostModel:
    """Fit k1..k4 from a profile CSV; the first util table becomes the UtilCurve."""
    batch, util = read_profile(path)
    if "attention" not in batch or "expert" not in batch:
        raise ConfigError(f"{path}: needs attention and expert rows")
    fa = calibrate(batch["attention"], "attention")
    fe = calibrate(batch["expert"], "expert")
    curve = UtilCurve.from_points(next(iter(util.values()))) if util else UtilCurve()
    beta = None if seq_len is None else fa.slope
    return CostModel(k1=fa.slope, k2=fa.intercept, k3=fe.slope, k4=fe.intercept,
                     alpha=0.0, beta=beta, util_curve=curve)
