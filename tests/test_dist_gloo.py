"""World-size-2 tests of the multi-GPU host logic on CPU (gloo backend)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_23317_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = shard.rank_tasks(rank, world, 6)
        # each rank "computes" a per-task output that depends only on the global task id
        out = torch.stack([torch.full((4,), float(t)) for t in mine])
        g = shard.gather_outputs(out)
        slowest = shard.max_over_ranks(1.5 + rank, "cpu")
        q.put((rank, mine, g.tolist(), slowest))
    finally:
        dist.destroy_process_group()


def test_two_rank_gather_and_max_over_ranks():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == list(range(0, 6)) and res[1][1] == list(range(6, 12))
    for _, _, g, slowest in res:
        assert slowest == 2.5                     # max over ranks
        flat = [row[0] for rk in g for row in rk]
        assert flat == [float(t) for t in range(12)]   # every task gathered exactly once, in rank order


def test_lpt_assignment_is_deterministic_and_balanced():
    import cfd_inputs as ci
    cfg = ci.CONFIGS["c640"]
    ks = [k for g in range(8) for k in ci.multi48_group_ks(g)]
    costs = [shard.task_cost(cfg.n_coarse + 3 * k, cfg.d_model, cfg.n_layers) for k in ks]
    a = shard.lpt_assign(costs, 8)
    assert a == shard.lpt_assign(costs, 8)
    assert sorted(i for r in a for i in r) == list(range(48))
    assert shard.imbalance(costs, a) < 1.05
    # degenerate: one rank gets everything
    assert shard.lpt_assign(costs, 1) == [list(range(48))]
