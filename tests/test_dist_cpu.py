"""Multi-process host logic on CPU (gloo, world_size 2): IPC-handle exchange,
role assignment and plan structs are identical on every rank."""

import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2504_02263_b200 import runtime
    from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    blob = bytes([rank]) * 64
    got = runtime.exchange_blobs(blob)
    assert got == [bytes([r]) * 64 for r in range(world)]
    plan = DeploymentPlan(n_a=1, n_e=1, m=2, b_a=64)
    model = as_model_spec("tiny")
    ps = runtime.make_plan_struct(model, plan)
    role = plan.role_of(rank)
    rec = [ps.world, ps.n_a, ps.n_e, ps.attn_ranks[0], ps.expert_ranks[0], ps.hidden, ps.inter,
           ps.experts, ps.topk, ps.max_tokens, ps.slots]
    all_rec = runtime.exchange_blobs(repr((rec, role)).encode())
    with open(os.path.join(outdir, f"r{rank}.txt"), "w") as fh:
        fh.write("\n".join(b.decode() for b in all_rec))
    dist.destroy_process_group()


def test_gloo_world2_exchange(tmp_path):
    port = _port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    a = (tmp_path / "r0.txt").read_text().splitlines()
    b = (tmp_path / "r1.txt").read_text().splitlines()
    assert a == b
    assert "'attention'" in a[0] and "'expert'" in a[1]
    assert a[0].startswith("([2, 1, 1, 0, 1, 512, 1536, 8, 2, 64, 2]")


def test_plan_struct_roles_for_bench_splits():
    from paper_2504_02263_b200 import runtime
    from paper_2504_02263_b200.config import DeploymentPlan, as_model_spec

    m = as_model_spec("mixtral-8x22b")
    for n_a, n_e, colo in ((1, 1, True), (1, 1, False), (3, 1, False), (6, 2, False)):
        p = DeploymentPlan(n_a=n_a, n_e=n_e, m=3, b_a=1024, colocated=colo)
        s = runtime.make_plan_struct(m, p)
        assert s.world == p.world
        assert list(s.attn_ranks[:n_a]) == p.attention_ranks()
        assert list(s.expert_ranks[:n_e]) == p.expert_ranks()
    with pytest.raises(ValueError):
        runtime.make_plan_struct(m, DeploymentPlan(n_a=8, n_e=8))  # 16 ranks > 8 per box
