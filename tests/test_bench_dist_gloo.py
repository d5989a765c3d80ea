"""bench.py's multi-GPU host path at world size 2 on CPU (gloo): the multi48 task sharding
(strong / weak, balanced groups / LPT stress mix), and the rank -> all_gather -> rank-0 oracle
check of sampled task outputs (bench.gather_and_check, the code the GPU run executes after
its timed region).  The per-task "GPU outputs" here are the oracle's own, so a correct gather
passes with zero error; a perturbed rank must fail the check."""
import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import cfd_inputs as ci


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_multi48_sharding_strong_weak_and_lpt():
    for world in (1, 2, 4, 8):
        strong = [bench.Work(bench.parse(["--workload", "multi48"]), r, world) for r in range(world)]
        ids = sorted(i for w in strong for i in w.ids)
        assert ids == list(range(48)) and all(len(w.ids) == 48 // world for w in strong)
        assert strong[0].frames_total == 48 and strong[0].scaling == "strong"
        # balanced groups: every rank holds whole groups of 6 with the same token total
        tok = {sum(w.counts) for w in strong}
        assert len(tok) == 1 and all(len(w.ids) % 6 == 0 for w in strong)
        weak = [bench.Work(bench.parse(["--workload", "multi48", "--scaling", "weak"]), r, world) for r in range(world)]
        assert weak[0].frames_total == 48 * world and all(len(w.ids) == 48 for w in weak)
        assert sorted(i for w in weak for i in w.ids) == list(range(48 * world))
        lpt = [bench.Work(bench.parse(["--workload", "multi48", "--mix", "s348"]), r, world) for r in range(world)]
        assert sorted(i for w in lpt for i in w.ids) == list(range(48))
        assert lpt[0].note["imbalance_max_over_mean"] < (1.1 if world < 8 else 1.35)
    with pytest.raises(SystemExit):
        bench.Work(bench.parse(["--workload", "multi48"]), 0, 5)


def _fake_full(work, corrupt):
    """A stand-in for the bench's single-lane encoder outputs: packed refined tokens, scores
    and cu_seqlens of the rank's tasks, the sampled tasks filled with the oracle's values."""
    import oracle as O
    cfg = work.cfg
    w = work.weights
    cu = np.concatenate([[0], np.cumsum(work.counts)]).astype(np.int32)
    y = torch.zeros(int(cu[-1]), cfg.d_model)
    scores = torch.zeros(len(work.ids), cfg.n_coarse)
    for i in bench.check_sample(work):
        img = ci.make_frame(cfg.img_h, cfg.img_w, ci.frame_seed(work.ids[i], 0))
        oc = O.coarse_encode(cfg, w, [img])[0]
        s32 = oc["scores"].astype(np.float32)
        rr = O.refine_encode(cfg, w, img, oc["x0"], O.select_topk(s32, work.ks[i]))
        y[cu[i]:cu[i + 1]] = torch.from_numpy(rr["y"]).float() + (0.1 if corrupt else 0.0)
        scores[i] = torch.from_numpy(s32)
    return types.SimpleNamespace(ro={"y": y, "cu_seqlens": torch.from_numpy(cu)}, co={"scores": scores})


def _worker(rank, world, port, corrupt_rank, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.set_num_threads(2)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        args = bench.parse(["--workload", "multi48", "--gpus", str(world)])
        work = bench.Work(args, rank, world)
        work.weights = ci.make_weights(work.cfg, seed=0)
        full = _fake_full(work, corrupt=(rank == corrupt_rank))
        res = bench.gather_and_check(args, work, full, rank, world, "cpu")
        q.put((rank, work.ids, res))
    finally:
        dist.destroy_process_group()


def _run(corrupt_rank):
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, corrupt_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.slow
def test_two_rank_gather_and_oracle_check():
    res = _run(corrupt_rank=-1)
    (r0, ids0, chk), (r1, ids1, none) = res
    assert none is None and ids0 == list(range(24)) and ids1 == list(range(24, 48))
    assert chk["pass"] and chk["ranks_checked"] == [0, 1] and chk["tasks_checked"] == 4
    assert chk["max_rel_l2"] < 1e-6 and chk["gathered_via"] == "gloo all_gather"
    # the gathered global ids are the sampled tasks of each rank
    assert {t[1] for t in chk["tasks"] if t[0] == 1} <= set(ids1)
    bad = _run(corrupt_rank=1)[0][2]
    assert not bad["pass"] and bad["max_abs"] >= 0.1 - 1e-6
