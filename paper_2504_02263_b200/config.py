"""Layer configuration and deployment plan for the disaggregated MoE decode step.

Drop-in for the reference's configuration API (``moeplan.catalog``,
/root/reference/pkg/src/moeplan/catalog.py).  The names, field order, defaults,
validation rules, error type and error texts follow that module so code written
against ``moeplan.catalog`` works unchanged:

* ``GpuSpec``       catalog.py:26-57     ``Catalog``         catalog.py:60-92
* ``MoeModelSpec``  catalog.py:95-124    ``WorkloadSpec``    catalog.py:127-142
* ``SearchLimits``  catalog.py:148-161   ``builtin_*``       catalog.py:164-191
* ``resolve_model`` catalog.py:194-202   ``ConfigBundle``    catalog.py:205-209
* ``config_from_dict`` / ``load_config`` / ``config_to_dict`` / ``save_config``
  catalog.py:230-290

Additions (additive only; a reference config file loads unchanged):

* a ``b200`` catalog entry carrying this pool's measured peaks (not in the
  builtin table, so ``builtin_catalog()`` stays identical to the reference);
* an optional top-level ``plan`` section -> ``DeploymentPlan`` with the SPEC's
  role vocabulary (``tp_a, tp_e, n_a, m, B``) plus ``n_e`` (expert
  GPUs) and ``b_a`` (tokens per attention GPU per micro-batch).  It is returned
  by :func:`load_plan` / :func:`plan_from_dict`; ``config_from_dict`` keeps the
  reference's four-key schema and return type.
"""

from __future__ import annotations

import json
from collections.abc import Mapping
from dataclasses import asdict, dataclass, fields
from pathlib import Path
from typing import Any, Iterator, NamedTuple

GB = 1e9
GBPS = 1e9
TFLOPS = 1e12

_NODE_SIZES = (1, 2, 4, 8)
_COST_METRICS = ("price", "power")
_TOP_KEYS = ("hardware", "model", "workload", "limits")

# Reference default: one 200 Gb/s NIC per GPU (catalog.py:17-19).
DEFAULT_NET_BANDWIDTH = 25 * GBPS
# NVLink 5 through NVSwitch, per GPU per direction (nominal).
NVLINK5_BANDWIDTH = 900 * GBPS


class ConfigError(ValueError):
    """Malformed or invalid configuration input (catalog.py:22-23)."""


def _positive(owner: str, obj, names) -> None:
    for attr in names:
        if not getattr(obj, attr) > 0:
            raise ConfigError(f"{owner}: {attr} must be > 0")


# --------------------------------------------------------------------------- #
# Hardware
# --------------------------------------------------------------------------- #
@dataclass(frozen=True)
class GpuSpec:
    """Accelerator entry (catalog.py:26-57): SI units, relative price."""

    name: str
    price: float
    mem_capacity: float
    mem_bandwidth: float
    compute: float
    net_bandwidth_per_gpu: float = DEFAULT_NET_BANDWIDTH
    max_power: float | None = None
    max_gpus_per_node: int = 8

    def __post_init__(self):
        if not self.name:
            raise ConfigError("gpu: name must be non-empty")
        _positive(f"gpu {self.name!r}", self,
                  ("price", "mem_capacity", "mem_bandwidth", "compute",
                   "net_bandwidth_per_gpu"))
        if self.max_power is not None and not self.max_power > 0:
            raise ConfigError(f"gpu {self.name!r}: max_power must be > 0 or null")
        if self.max_gpus_per_node not in _NODE_SIZES:
            raise ConfigError(
                f"gpu {self.name!r}: max_gpus_per_node must be one of {_NODE_SIZES}")


class Catalog(Mapping):
    """Case-insensitive, immutable name -> GpuSpec map (catalog.py:60-92)."""

    def __init__(self, gpus):
        table: dict[str, GpuSpec] = {}
        seen: set[str] = set()
        for gpu in gpus:
            key = gpu.name.lower()
            if key in seen:
                raise ConfigError(f"catalog: duplicate gpu name {gpu.name!r}")
            seen.add(key)
            table[gpu.name] = gpu
        if not table:
            raise ConfigError("catalog: at least one gpu entry required")
        self._entries = table

    def __getitem__(self, name: str) -> GpuSpec:
        hit = self._entries.get(name)
        if hit is not None:
            return hit
        want = name.lower()
        for key, gpu in self._entries.items():
            if key.lower() == want:
                return gpu
        raise KeyError(name)

    def __iter__(self) -> Iterator[str]:
        return iter(self._entries)

    def __len__(self) -> int:
        return len(self._entries)

    def __eq__(self, other) -> bool:
        return isinstance(other, Catalog) and self._entries == other._entries

    def __repr__(self) -> str:
        return f"Catalog({list(self._entries)})"


def builtin_catalog() -> Catalog:
    """The reference's Table-4 catalog, values verbatim (catalog.py:164-177)."""
    rows = (
        # name     price  mem GB  GB/s    TFLOPS  power
        ("L20",    1.00,  48,     864,    119.5,  None),
        ("H800",   5.28,  80,     3430.4, 989,    None),
        ("A800",   2.26,  80,     2039,   312,    None),
        ("H20",    1.85,  96,     4096,   148,    500.0),
        ("L40S",   1.08,  48,     864,    362,    350.0),
    )
    gpus = []
    for name, price, cap, bw, flops, power in rows:
        kw = {} if power is None else {"max_power": power}
        gpus.append(GpuSpec(name, price=price, mem_capacity=cap * GB,
                            mem_bandwidth=bw * GB, compute=flops * TFLOPS, **kw))
    return Catalog(gpus)


def b200_gpu(peaks: Mapping | None = None) -> GpuSpec:
    """A B200 entry.  ``peaks`` is MEASURED_PEAKS.json (hbm_gbs, bf16_tflops);
    without it the nominal HGX figures are used.  Price is relative (unknown
    market price; 1.0 placeholder), power 1000 W, NVLink 5 per direction."""
    hbm = float(peaks["hbm_gbs"]) if peaks and "hbm_gbs" in peaks else 7700.0
    tf = float(peaks["bf16_tflops"]) if peaks and "bf16_tflops" in peaks else 2250.0
    return GpuSpec("B200", price=1.0, mem_capacity=180 * GB,
                   mem_bandwidth=hbm * GB, compute=tf * TFLOPS,
                   net_bandwidth_per_gpu=NVLINK5_BANDWIDTH, max_power=1000.0,
                   max_gpus_per_node=8)


# --------------------------------------------------------------------------- #
# Model / workload / limits
# --------------------------------------------------------------------------- #
@dataclass(frozen=True)
class MoeModelSpec:
    """MoE layer parameters (catalog.py:95-124).  ``hidden`` = h,
    ``intermediate`` = h', ``experts`` = E, ``topk`` = K."""

    name: str
    layers: int
    hidden: int
    intermediate: int
    experts: int
    topk: int
    gqa_group: int = 8
    bytes_per_param: int = 2

    def __post_init__(self):
        _positive(f"model {self.name!r}", self, ("layers", "hidden", "intermediate"))
        if not 1 <= self.topk <= self.experts:
            raise ConfigError(
                f"model {self.name!r}: K out of range (1 <= topk <= experts)")
        if self.gqa_group < 1:
            raise ConfigError(f"model {self.name!r}: gqa_group must be >= 1")
        if self.bytes_per_param < 1:
            raise ConfigError(f"model {self.name!r}: bytes_per_param must be >= 1")


@dataclass(frozen=True)
class WorkloadSpec:
    """Traffic statistics and TBT SLO (catalog.py:127-142)."""

    avg_seq_len: int = 730
    slo_tbt: float = 0.150
    input_len_median: int = 571
    output_len_median: int = 159

    def __post_init__(self):
        if not self.avg_seq_len > 0:
            raise ConfigError("workload: avg_seq_len must be > 0")
        if not self.slo_tbt > 0:
            raise ConfigError("workload: slo_tbt must be > 0")
        if min(self.input_len_median, self.output_len_median) < 0:
            raise ConfigError("workload: median lengths must be >= 0")


@dataclass(frozen=True)
class SearchLimits:
    """Planner search bounds (catalog.py:148-161)."""

    max_microbatches: int = 4
    cost_metric: str = "price"

    def __post_init__(self):
        if self.max_microbatches < 3:
            raise ConfigError("limits: max_microbatches must be >= 3")
        if self.cost_metric not in _COST_METRICS:
            raise ConfigError(f"limits: cost_metric must be one of {_COST_METRICS}")


def builtin_models() -> dict[str, MoeModelSpec]:
    """Table-5 models, verbatim (catalog.py:180-191)."""
    specs = (
        MoeModelSpec("Mixtral-8x22B", layers=56, hidden=6144,
                     intermediate=16384, experts=8, topk=2),
        MoeModelSpec("DBRX", layers=40, hidden=6144,
                     intermediate=10752, experts=16, topk=4),
        MoeModelSpec("Scaled-MoE", layers=48, hidden=8192,
                     intermediate=8192, experts=32, topk=4),
    )
    return {m.name: m for m in specs}


def resolve_model(name: str) -> MoeModelSpec:
    """Case-insensitive builtin lookup (catalog.py:194-202)."""
    models = builtin_models()
    want = name.lower()
    for key, spec in models.items():
        if key.lower() == want:
            return spec
    raise ConfigError(f"model: unknown builtin {name!r} (choices: {sorted(models)})")


# The BASELINE.json layer shapes that are not reference builtins; their
# intermediate sizes are pinned in SURVEY.md §8 (public model configs).
BENCH_SHAPES: dict[str, MoeModelSpec] = {
    "tiny": MoeModelSpec("tiny", layers=1, hidden=512, intermediate=1536,
                         experts=8, topk=2),
    "mixtral-8x7b": MoeModelSpec("Mixtral-8x7B", layers=32, hidden=4096,
                                 intermediate=14336, experts=8, topk=2),
    "mixtral-8x22b": builtin_models()["Mixtral-8x22B"],
    "dbrx": builtin_models()["DBRX"],
    "deepseek-v3": MoeModelSpec("DeepSeek-V3-shape", layers=61, hidden=7168,
                                intermediate=2048, experts=256, topk=8),
}


def as_model_spec(obj) -> MoeModelSpec:
    """Accept a MoeModelSpec, a duck-typed ``moeplan.catalog.MoeModelSpec``, a
    builtin/bench name or a dict."""
    if isinstance(obj, MoeModelSpec):
        return obj
    if isinstance(obj, str):
        key = obj.lower()
        if key in BENCH_SHAPES:
            return BENCH_SHAPES[key]
        return resolve_model(obj)
    if isinstance(obj, Mapping):
        return _build(MoeModelSpec, dict(obj), "model")
    try:
        return MoeModelSpec(**{f.name: getattr(obj, f.name) for f in fields(MoeModelSpec)})
    except AttributeError as exc:
        raise ConfigError(f"model: not a MoeModelSpec-like object ({exc})") from exc


# --------------------------------------------------------------------------- #
# Config documents (catalog.py:205-290)
# --------------------------------------------------------------------------- #
class ConfigBundle(NamedTuple):
    catalog: Catalog
    model: MoeModelSpec
    workload: WorkloadSpec
    limits: SearchLimits


def _check_keys(mapping, allowed, section: str) -> None:
    unknown = [k for k in mapping if k not in allowed]
    if unknown:
        raise ConfigError(f"{section}: unknown key {unknown[0]!r}")


def _build(cls, raw: dict, section: str):
    _check_keys(raw, tuple(f.name for f in fields(cls)), section)
    try:
        return cls(**raw)
    except TypeError as exc:
        raise ConfigError(f"{section}: {exc}") from exc


def _bundle(doc: dict) -> ConfigBundle:
    hardware = doc.get("hardware")
    if hardware is None:
        catalog = builtin_catalog()
    elif isinstance(hardware, list) and hardware:
        catalog = Catalog([_build(GpuSpec, g, "hardware entry") for g in hardware])
    else:
        raise ConfigError("hardware: must be a non-empty array")

    if "model" not in doc or doc["model"] is None:
        raise ConfigError("config: missing required key 'model'")
    raw_model = doc["model"]
    if isinstance(raw_model, str):
        model = resolve_model(raw_model)
    elif isinstance(raw_model, dict):
        model = _build(MoeModelSpec, raw_model, "model")
    else:
        raise ConfigError("model: must be a builtin name or an object")

    workload = _build(WorkloadSpec, doc.get("workload", {}), "workload")
    limits = _build(SearchLimits, doc.get("limits", {}), "limits")
    return ConfigBundle(catalog, model, workload, limits)


def config_from_dict(doc: dict) -> ConfigBundle:
    """Validate a parsed config document (catalog.py:230-256)."""
    if not isinstance(doc, dict):
        raise ConfigError("config: top level must be a JSON object")
    _check_keys(doc, _TOP_KEYS, "config")
    return _bundle(doc)


def _read_json(path: Path) -> Any:
    try:
        text = path.read_text()
    except OSError as exc:
        raise ConfigError(f"{path}: {exc}") from exc
    try:
        return json.loads(text)
    except json.JSONDecodeError as exc:
        raise ConfigError(
            f"{path}: parse error at line {exc.lineno} column {exc.colno}: {exc.msg}"
        ) from exc


def load_config(path) -> ConfigBundle:
    """Load and validate a JSON config file (catalog.py:259-276)."""
    return config_from_dict(_read_json(Path(path)))


def config_to_dict(bundle: ConfigBundle) -> dict[str, Any]:
    """Serialize back to the file schema (catalog.py:279-286)."""
    return {
        "hardware": [asdict(g) for g in bundle.catalog.values()],
        "model": asdict(bundle.model),
        "workload": asdict(bundle.workload),
        "limits": asdict(bundle.limits),
    }


def save_config(bundle: ConfigBundle, path) -> None:
    Path(path).write_text(json.dumps(config_to_dict(bundle), indent=2) + "\n")


# --------------------------------------------------------------------------- #
# Deployment plan (additive ``plan`` section)
# --------------------------------------------------------------------------- #
@dataclass(frozen=True)
class DeploymentPlan:
    """Roles of one decode deployment on a single NVSwitch box.

    SPEC.md:311 vocabulary: ``tp_a``, ``tp_e``, ``n_a``
    attention GPUs (data-parallel replicas), ``m`` micro-batches
    (ping-pong), ``B`` = global batch per micro-batch
    (= n_a * b_a).  Added: ``n_e`` expert GPUs and ``b_a``.  Expert GPUs form
    n_e / tp_e expert nodes of tp_e GPUs (the paper's expert node = one expert
    over tp_e GPUs); expert e lives on node
    e // (E / nodes), contiguous blocks, and every GPU of the node holds h'/tp_e
    features of each of the node's experts (tensor parallel over h'; the
    combine sums the tp_e partial outputs).  Attention GPUs form n_a / tp_a
    attention nodes of tp_a GPUs (tensor parallel over heads, PAPER.md:192,
    441-443): every GPU keeps its own b_a-token shard (its M2N batch) and
    1/tp_a of the heads; the QKV GEMM all-gathers the node's shards over
    NVLink and the O projection reduce-scatters them back (attn_tp.cu).
    ``colocated`` puts both roles on
    every GPU (the 1-GPU report point, and the DeepSeek-shaped 8->8 case); then
    n_a == n_e == world size and tp_e == 1.
    """

    n_a: int = 1
    n_e: int = 1
    m: int = 1
    b_a: int = 64
    tp_a: int = 1
    tp_e: int = 1
    colocated: bool = False

    def __post_init__(self):
        _positive("plan", self, ("n_a", "n_e", "m", "b_a"))
        if self.tp_a < 1 or self.n_a % self.tp_a or self.tp_a > 8:
            raise ConfigError(f"plan: tp_a ({self.tp_a}) must divide n_a ({self.n_a}) and be <= 8")
        if self.tp_e < 1 or self.n_e % self.tp_e:
            raise ConfigError(f"plan: tp_e ({self.tp_e}) must divide n_e ({self.n_e})")
        if self.colocated and self.n_a != self.n_e:
            raise ConfigError("plan: colocated plans need n_a == n_e")
        if self.colocated and self.tp_e != 1:
            raise ConfigError("plan: expert TP (tp_e > 1) needs separate expert GPUs")

    @property
    def B(self) -> int:  # noqa: N802 - SPEC name
        return self.n_a * self.b_a

    @property
    def world(self) -> int:
        return self.n_a if self.colocated else self.n_a + self.n_e

    def attention_ranks(self) -> list[int]:
        return list(range(self.n_a))

    def expert_ranks(self) -> list[int]:
        if self.colocated:
            return list(range(self.n_e))
        return list(range(self.n_a, self.n_a + self.n_e))

    def role_of(self, rank: int) -> str:
        if not 0 <= rank < self.world:
            raise ConfigError(f"plan: rank {rank} outside world {self.world}")
        if self.colocated:
            return "both"
        return "attention" if rank < self.n_a else "expert"

    @property
    def expert_nodes(self) -> int:
        return self.n_e // self.tp_e

    def check_model(self, model: MoeModelSpec) -> None:
        if model.experts % self.expert_nodes:
            raise ConfigError(
                f"plan: experts ({model.experts}) must divide evenly over the {self.expert_nodes} expert nodes")
        if model.intermediate % (128 * self.tp_e):
            raise ConfigError(f"plan: intermediate ({model.intermediate}) must split into tp_e multiples of 128")

    def experts_per_gpu(self, model: MoeModelSpec) -> int:
        """Experts whose (TP slice of the) weights every expert GPU holds."""
        self.check_model(model)
        return model.experts // self.expert_nodes


def plan_from_dict(raw: dict) -> DeploymentPlan:
    return _build(DeploymentPlan, dict(raw), "plan")


def load_plan(path) -> tuple[ConfigBundle, DeploymentPlan]:
    """Load a config file that may carry the additive ``plan`` key."""
    doc = _read_json(Path(path))
    if not isinstance(doc, dict):
        raise ConfigError("config: top level must be a JSON object")
    _check_keys(doc, _TOP_KEYS + ("plan", "plan_info"), "config")
    plan = plan_from_dict(doc.get("plan", {}))
    bundle = _bundle({k: v for k, v in doc.items() if k not in ("plan", "plan_info")})
    plan.check_model(bundle.model)
    return bundle, plan


def save_plan(bundle: ConfigBundle, plan: DeploymentPlan, path, extra: dict | None = None) -> None:
    """Write a config file with the additive ``plan`` section (the planner's
    output, read back by ``load_plan``).  ``extra`` keys (e.g. the planner's
    predicted times) go under ``plan_info``, which ``load_plan`` ignores."""
    plan.check_model(bundle.model)
    doc = config_to_dict(bundle)
    doc["plan"] = asdict(plan)
    text = json.dumps(doc, indent=2) + "\n"
    if extra:
        doc2 = dict(doc)
        doc2["plan_info"] = extra
        text = json.dumps(doc2, indent=2, default=float) + "\n"
    Path(path).write_text(text)
