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


# ---------------------------------------------------------------------------------------------------
# Mode 2: one large shape, query blocks sharded across ranks.
# Every rank builds the same plan from the same coordinates (deterministic, no communication); rank r
# owns the contiguous query-block range [q_begin, q_end) of plan order (balanced by token count, the
# cost of a query block being ~ its rows x the compressed keys of the shape). K/V are all-gathered,
# the library computes only the owned rows, and the dK/dV partials are summed across ranks.
# ---------------------------------------------------------------------------------------------------
def balanced_q_ranges(q_offsets, world: int):
    """Split query blocks [0, n_q) into `world` contiguous ranges with ~equal token counts.
    q_offsets: the plan's SSA_LEVEL_Q offsets (length n_q + 1, tokens)."""
    import numpy as np
    off = np.asarray(q_offsets, dtype=np.int64)
    n_q, total = len(off) - 1, int(off[-1])
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        cuts.append(int(np.clip(np.searchsorted(off, target, side="left"), cuts[-1], n_q)))
    cuts.append(n_q)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def ssa_step_sharded(plan, cfg, q_sorted, k_local, v_local, gates_sorted, dout_sorted, tok_ranges, rank, group=None):
    """Forward + backward of one shape sharded by query blocks (NCCL / any torch.distributed group).

    Inputs are in plan (block-sorted) order. k_local / v_local hold this rank's token range
    tok_ranges[rank] (padded to the largest range); q / gates / dout are full-size buffers of which only
    the owned rows are read. Returns (out, dq, dk_local, dv_local, dgates): out / dq / dgates are valid on
    the owned rows, dk_local / dv_local are this rank's tokens' complete gradients.
    Collectives: one all-gather of K and V (forward), one all-reduce of the dK / dV partials (backward).
    """
    import dataclasses
    import torch
    import torch.distributed as dist
    from . import ssa
    world = len(tok_ranges)
    pad = max(b - a for a, b in tok_ranges)
    shape = (world * pad,) + tuple(k_local.shape[1:])
    k_all = torch.empty(shape, dtype=k_local.dtype, device=k_local.device)
    v_all = torch.empty_like(k_all)
    if world == 1:
        k_all.copy_(k_local)
        v_all.copy_(v_local)
    else:
        dist.all_gather_into_tensor(k_all, k_local.contiguous(), group=group)
        dist.all_gather_into_tensor(v_all, v_local.contiguous(), group=group)
    k = torch.cat([k_all[r * pad: r * pad + (b - a)] for r, (a, b) in enumerate(tok_ranges)])
    v = torch.cat([v_all[r * pad: r * pad + (b - a)] for r, (a, b) in enumerate(tok_ranges)])
    qo = plan.offsets(ssa.LEVEL_Q).cpu().tolist()
    qb = [qo.index(a) for a, _ in tok_ranges] + [len(qo) - 1]
    c2 = dataclasses.replace(cfg, flags=cfg.flags | ssa.SSA_INPUT_SORTED | ssa.SSA_KV_GRAD_FP32,
                             q_begin=qb[rank], q_end=qb[rank + 1])
    out, saved = ssa.ssa_forward(plan, c2, q_sorted, k, v, gates_sorted)
    dq, dk, dv, dg = ssa.ssa_backward(plan, c2, saved, q_sorted, k, v, gates_sorted, dout_sorted)
    if world > 1:
        dist.all_reduce(dk, group=group)      # fp32 partials (SSA_KV_GRAD_FP32)
        dist.all_reduce(dv, group=group)
    a, b = tok_ranges[rank]
    return out, dq, dk[a:b].to(k_local.dtype), dv[a:b].to(k_local.dtype), dg
