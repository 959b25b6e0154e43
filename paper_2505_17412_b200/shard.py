"""Host-side multi-GPU orchestration for SSA (no data-path collective).

SSA has no parameters and the shapes of a batch never interact (SURVEY §8e mode 1), so N GPUs process
disjoint subsets of the shapes; torch.distributed is used only for the timing barrier and the
max-over-ranks reduction. Shapes are dealt by LPT on a cost model ~ n_tokens^2 (the compression
branch dominates and is quadratic in the token count).
"""
from __future__ import annotations


def lpt_assign(costs, world: int):
    """Longest-processing-time assignment: returns one list of item indices per rank (deterministic:
    ties broken by item index, then by rank index)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    loads = [0.0] * world
    out = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda j: (loads[j], j))
        loads[r] += costs[i]
        out[r].append(i)
    return [sorted(x) for x in out]


def rank_items(n_tokens, rank: int, world: int):
    """Indices of the shapes rank `rank` processes (cost = n_tokens^2)."""
    if world <= 1:
        return list(range(len(n_tokens)))
    return lpt_assign([float(n) ** 2 for n in n_tokens], world)[rank]


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. a CUDA-event time) over the process group."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
