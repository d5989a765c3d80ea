"""Multi-GPU host logic: camera tasks shard across ranks with no collective on the
hot path (tasks are independent, attention is per task, R11).

One process per GPU.  Collectives are used only around the timed region: the
max-over-ranks step time and the gather of per-task outputs for checking (NCCL on
GPUs; the same functions run on gloo/CPU in tests/test_dist_gloo.py).
"""
from __future__ import annotations

from typing import List, Sequence

import torch


def rank_tasks(rank: int, world: int, per_rank: int) -> List[int]:
    """Weak scaling: rank r owns the contiguous global task ids [r*per_rank, (r+1)*per_rank)."""
    assert 0 <= rank < world
    return list(range(rank * per_rank, (rank + 1) * per_rank))


def task_cost(n_tokens: int, d: int, n_layers: int) -> int:
    """Predicted encoder cost of one task: L * (24 d^2 N + 4 d N^2) FLOPs (linear + attention)."""
    return n_layers * (24 * d * d * n_tokens + 4 * d * n_tokens * n_tokens)


def lpt_assign(costs: Sequence[int], world: int) -> List[List[int]]:
    """Longest-processing-time-first assignment of tasks to ranks (deterministic:
    ties broken by lower task id, then lower rank).  Returns task ids per rank, each
    list ascending."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0] * world
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += costs[i]
    return [sorted(x) for x in out]


def imbalance(costs: Sequence[int], assignment: Sequence[Sequence[int]]) -> float:
    loads = [sum(costs[i] for i in a) for a in assignment]
    mean = sum(loads) / len(loads)
    return max(loads) / mean if mean else 1.0


def max_over_ranks(value: float, device) -> float:
    """Max of a per-rank scalar (timing is reported as the slowest rank)."""
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_outputs(t: torch.Tensor) -> torch.Tensor:
    """All-gather a fixed-shape per-rank tensor -> [world, *shape] (outside timing)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return t[None]
    out = torch.empty((dist.get_world_size(), *t.shape), dtype=t.dtype, device=t.device)
    if t.is_cuda:
        dist.all_gather_into_tensor(out, t.contiguous())
    else:
        dist.all_gather(list(out.unbind(0)), t.contiguous())
    return out
