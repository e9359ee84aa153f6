"""Multi-rank combine on CPU: world_size 2 over gloo.

Component values come from the CPU oracle (the GPU is not needed to test
the partition / all-gather / ordered-sum logic); the distributed result
must be bitwise equal to the single-rank plan-order sum.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1707_09598_b200 import configs
from paper_1707_09598_b200.distributed import (component_cost_model, ordered_combine, plan_partition)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _values(name, indices, coefs_all, pts):
    from oracle import oracle as O
    from paper_1707_09598_b200.scheduler import make_spec

    cfg = configs.get_config(name)
    orc = O.Oracle(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points), threads=1)
    return np.stack([orc.combine_points(pts, coefs=coefs_all, comp=i) for i in indices]) if indices else \
        np.zeros((0, pts.shape[0]))


def _worker(rank, world, port, name, coefs_all, pts, out_path):
    import torch.distributed as dist

    from paper_1707_09598_b200.distributed import combine_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = configs.get_config(name)
    vals = combine_distributed(cfg.plan, pts.shape[0], lambda idx: _values(name, idx, coefs_all, pts),
                               cfg.problem.degree)
    np.save(f"{out_path}.{rank}.npy", vals)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg1", "cfg3"])
def test_two_rank_combine_bitwise(tmp_path, name):
    from oracle import oracle as O
    from paper_1707_09598_b200.scheduler import make_spec

    cfg = configs.get_config(name)
    orc = O.Oracle(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
    coefs = orc.run_plan(O.SOLVER_DIRECT)
    pts = cfg.points(300)
    single = ordered_combine(cfg.plan, _values(name, list(range(len(cfg.plan))), coefs, pts))
    # the single-rank ordered sum equals the oracle's own plan-order combine
    assert np.array_equal(single, orc.combine_points(pts, coefs=coefs))
    world, port, out = 2, _free_port(), str(tmp_path / "vals")
    mp.spawn(_worker, args=(world, port, name, coefs, pts, out), nprocs=world, join=True)
    for r in range(world):
        assert np.array_equal(np.load(f"{out}.{r}.npy"), single)


def test_partition_is_lpt_and_complete():
    cfg = configs.get_config("cfg5")
    for world in (1, 2, 4, 8):
        parts = plan_partition(cfg.plan, world, cfg.problem.degree)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(cfg.plan)))
        cost = component_cost_model(cfg.plan.terms, cfg.problem.degree, 3)
        loads = [cost[p].sum() for p in parts]
        assert max(loads) <= cost.sum() / world + cost.max() + 1e-9   # LPT bound
