"""Config API is a drop-in for moeplan.catalog (catalog.py:95-290)."""

import json
import os
import sys

import pytest

from paper_2504_02263_b200 import config as C

REF_SRC = "/root/reference/pkg/src"


def test_builtin_models_verbatim():
    m = C.builtin_models()
    assert m["Mixtral-8x22B"] == C.MoeModelSpec("Mixtral-8x22B", 56, 6144, 16384, 8, 2)
    assert m["DBRX"].layers == 40 and m["DBRX"].experts == 16 and m["DBRX"].topk == 4
    assert m["Scaled-MoE"].experts == 32 and m["Scaled-MoE"].hidden == 8192


def test_builtin_catalog_verbatim():
    cat = C.builtin_catalog()
    assert cat["H20"].mem_bandwidth == 4096 * C.GB
    assert cat["L40S"].compute == 362 * C.TFLOPS
    assert cat["l20"].price == 1.00  # case-insensitive lookup
    assert cat["H20"].max_power == 500.0 and cat["A800"].max_power is None
    assert list(cat) == ["L20", "H800", "A800", "H20", "L40S"]


@pytest.mark.parametrize("kw,msg", [
    (dict(topk=0), "K out of range"),
    (dict(topk=9), "K out of range"),
    (dict(hidden=0), "hidden must be > 0"),
    (dict(gqa_group=0), "gqa_group must be >= 1"),
    (dict(bytes_per_param=0), "bytes_per_param must be >= 1"),
])
def test_model_validation(kw, msg):
    base = dict(name="m", layers=1, hidden=8, intermediate=8, experts=8, topk=2)
    base.update(kw)
    with pytest.raises(C.ConfigError, match=msg):
        C.MoeModelSpec(**base)


def test_loader_defaults_and_errors(tmp_path):
    b = C.config_from_dict({"model": "dbrx"})
    assert b.model.name == "DBRX" and b.workload.avg_seq_len == 730 and b.limits.max_microbatches == 4
    with pytest.raises(C.ConfigError, match="unknown key"):
        C.config_from_dict({"model": "dbrx", "bogus": 1})
    with pytest.raises(C.ConfigError, match="missing required key 'model'"):
        C.config_from_dict({})
    with pytest.raises(C.ConfigError, match="K out of range"):
        C.config_from_dict({"model": {"name": "x", "layers": 1, "hidden": 8, "intermediate": 8,
                                      "experts": 4, "topk": 0}})
    p = tmp_path / "bad.json"
    p.write_text('{"model": "dbrx",\n  oops}')
    with pytest.raises(C.ConfigError, match="parse error at line 2"):
        C.load_config(p)
    with pytest.raises(C.ConfigError, match="max_microbatches must be >= 3"):
        C.config_from_dict({"model": "dbrx", "limits": {"max_microbatches": 2}})


def test_round_trip(tmp_path):
    b = C.config_from_dict({"model": "Mixtral-8x22B", "workload": {"slo_tbt": 0.2}})
    p = tmp_path / "c.json"
    C.save_config(b, p)
    assert C.load_config(p) == b
    assert b.workload.slo_tbt == 0.2


def test_plan_section(tmp_path):
    p = tmp_path / "plan.json"
    p.write_text(json.dumps({"model": "Mixtral-8x22B", "plan": {"n_a": 6, "n_e": 2, "m": 3, "b_a": 1024}}))
    bundle, plan = C.load_plan(p)
    assert plan.B == 6144 and plan.world == 8
    assert plan.attention_ranks() == [0, 1, 2, 3, 4, 5] and plan.expert_ranks() == [6, 7]
    assert plan.role_of(0) == "attention" and plan.role_of(7) == "expert"
    assert plan.experts_per_gpu(bundle.model) == 4
    colo = C.DeploymentPlan(n_a=8, n_e=8, colocated=True)
    assert colo.world == 8 and colo.role_of(3) == "both"
    with pytest.raises(C.ConfigError):
        C.DeploymentPlan(n_a=1, n_e=3).check_model(bundle.model)  # 8 experts over 3 GPUs
    with pytest.raises(C.ConfigError):
        C.DeploymentPlan(tp_a=2)
    # the reference schema (no plan) still loads through load_config
    q = tmp_path / "ref.json"
    q.write_text(json.dumps({"model": "DBRX"}))
    assert C.load_config(q).model.name == "DBRX"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not mounted (GPU box)")
def test_matches_reference_moeplan():
    """Same builtins, same validation, objects interchangeable (duck typing)."""
    sys.path.insert(0, REF_SRC)
    try:
        from moeplan import catalog as R
    finally:
        sys.path.remove(REF_SRC)
    for name, spec in R.builtin_models().items():
        assert C.as_model_spec(spec) == C.builtin_models()[name]
    for name, g in R.builtin_catalog().items():
        ours = C.builtin_catalog()[name]
        assert [getattr(g, f) for f in g.__dataclass_fields__] == [getattr(ours, f) for f in g.__dataclass_fields__]
    doc = {"model": "dbrx", "workload": {"slo_tbt": 0.1}}
    assert R.config_to_dict(R.config_from_dict(doc)) == C.config_to_dict(C.config_from_dict(doc))
    for bad in ({"model": "dbrx", "x": 1}, {"model": {"name": "a", "layers": 1, "hidden": 1,
                                                         "intermediate": 1, "experts": 2, "topk": 3}}):
        with pytest.raises(ValueError) as e1:
            R.config_from_dict(bad)
        with pytest.raises(ValueError) as e2:
            C.config_from_dict(bad)
        assert str(e1.value) == str(e2.value)


def test_plan_expert_tp_validation():
    """Expert TP (tp_e): nodes of tp_e expert GPUs share their experts; tp_e
    must divide n_e, experts divide over the nodes, h' split in 128s, and
    co-located plans keep tp_e = 1."""
    m = C.as_model_spec("mixtral-8x22b")
    p = C.DeploymentPlan(n_a=2, n_e=4, tp_e=2)
    assert p.expert_nodes == 2 and p.experts_per_gpu(m) == 4 and p.world == 6
    assert p.expert_ranks() == [2, 3, 4, 5]
    with pytest.raises(C.ConfigError, match="tp_e"):
        C.DeploymentPlan(n_a=2, n_e=3, tp_e=2)
    with pytest.raises(C.ConfigError, match="expert TP"):
        C.DeploymentPlan(n_a=2, n_e=2, tp_e=2, colocated=True)
    assert C.DeploymentPlan(n_a=2, n_e=2, tp_a=2).tp_a == 2  # attention node of 2 GPUs
    with pytest.raises(C.ConfigError, match="tp_a"):
        C.DeploymentPlan(n_a=3, n_e=2, tp_a=2)
    with pytest.raises(C.ConfigError, match="tp_a"):
        C.DeploymentPlan(n_a=2, n_e=2, tp_a=0)
    with pytest.raises(C.ConfigError, match="divide evenly"):
        C.DeploymentPlan(n_a=1, n_e=6, tp_e=2).check_model(m)  # 3 nodes for 8 experts
    tiny = C.as_model_spec("tiny")  # h' = 1536 = 12 x 128: tp 4 -> 384 = 3 x 128
    C.DeploymentPlan(n_a=1, n_e=4, tp_e=4).check_model(tiny)
    with pytest.raises(C.ConfigError, match="intermediate"):
        C.DeploymentPlan(n_a=1, n_e=8, tp_e=8).check_model(tiny)  # 192 not a multiple of 128
