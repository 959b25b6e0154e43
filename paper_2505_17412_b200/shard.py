"""Host-side multi-GPU orchestration for SSA.

Mode 1 (batch of shapes): SSA has no parameters and the shapes of a batch never interact, so N GPUs
process disjoint subsets of the shapes with no data-path collective; torch.distributed is used only for
the timing barrier and the max-over-ranks reduction. Shapes are dealt by LPT on a cost model
~ n_tokens^2 (the compression branch dominates and is quadratic in the token count).
Mode 2 (one large shape): query blocks sharded over ranks (ssa_step_sharded) with the path's real
exchange steps: pooled-key all-reduce, K/V all-gather (overlapped with the compression branch) and the
dK/dV reduce-scatter.
Hybrid (C4 at scale): hybrid_plan splits the largest shapes of a batch over sub-groups of ranks.
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


def _backend(group):
    import torch.distributed as dist
    return dist.get_backend(group) if dist.is_initialized() else "none"


def all_gather_rows(full, local, tok_ranges, rank, group=None):
    """full[a_r:b_r] = rank r's `local` rows for every rank r (one padded all-gather; gloo groups stage
    through host memory). full: [N, ...] on local's device."""
    import torch
    import torch.distributed as dist
    world = len(tok_ranges)
    pad = max(b - a for a, b in tok_ranges)
    a, b = tok_ranges[rank]
    if world == 1:
        full[a:b].copy_(local)
        return full
    send = torch.zeros((pad,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    send[:b - a] = local
    if _backend(group) == "nccl":
        got = torch.empty((world * pad,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(got, send, group=group)
    else:
        parts = [torch.empty_like(send, device="cpu") for _ in range(world)]
        dist.all_gather(parts, send.cpu(), group=group)
        got = torch.cat(parts).to(local.device)
    for r, (x, y) in enumerate(tok_ranges):
        full[x:y] = got[r * pad: r * pad + (y - x)]
    return full


def reduce_scatter_rows(full, tok_ranges, rank, group=None):
    """Sum over ranks of full[a_r:b_r] for this rank's range (one padded reduce-scatter; gloo groups stage
    through host memory with an all-reduce)."""
    import torch
    import torch.distributed as dist
    world = len(tok_ranges)
    a, b = tok_ranges[rank]
    if world == 1:
        return full[a:b].clone()
    pad = max(y - x for x, y in tok_ranges)
    send = torch.zeros((world * pad,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
    for r, (x, y) in enumerate(tok_ranges):
        send[r * pad: r * pad + (y - x)] = full[x:y]
    if _backend(group) == "nccl":
        out = torch.empty((pad,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
        dist.reduce_scatter_tensor(out, send, group=group)
    else:
        h = send.cpu()
        dist.all_reduce(h, group=group)
        out = h[rank * pad:(rank + 1) * pad].to(full.device)
    return out[:b - a]


def all_reduce_sum(t, group=None):
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return t
    if _backend(group) == "nccl":
        dist.all_reduce(t, group=group)
    else:
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    return t


def shard_ranges(plan, world: int):
    """(query-block ranges, token ranges) of the `world` shards of one plan (every rank computes the
    same from the same plan)."""
    qo = plan.q_offsets_host()
    rng = balanced_q_ranges(qo, world)
    return rng, [(int(qo[a]), int(qo[b])) for a, b in rng]


def exchange_peer_pointers(k_loc, v_loc, rank, world, group=None):
    """One-sided K/V access: every rank exports its own K/V rows as CUDA IPC handles,
    all ranks exchange them, and each opens the others' (peer mappings: NVLink P2P on a multi-GPU node,
    a second mapping of the same memory when the ranks share one GPU). Returns (peer_k, peer_v, bases
    to close)."""
    import torch.distributed as dist
    from . import ssa
    mine = (ssa.ipc_export(k_loc), ssa.ipc_export(v_loc))
    allh = [None] * world
    if world > 1:
        dist.all_gather_object(allh, mine, group=group)
    else:
        allh = [mine]
    pk, pv, bases = [], [], []
    for r, ((hk, ok), (hv, ov)) in enumerate(allh):
        if r == rank:
            pk.append(k_loc.data_ptr())
            pv.append(v_loc.data_ptr())
            continue
        bk, p1 = ssa.ipc_open(hk, ok)
        bv, p2 = ssa.ipc_open(hv, ov)
        pk.append(p1)
        pv.append(p2)
        bases += [bk, bv]
    return pk, pv, bases


def ssa_step_sharded(plan, cfg, q_loc, k_loc, v_loc, gates_loc, dout_loc, rank, world, group=None,
                     comm_stream=None, q_ranges=None, exchange="allgather"):
    """Forward + backward of ONE shape with its query blocks sharded over `world` ranks (SURVEY §8e
    mode 2). Every rank built the same plan; rank r holds only its own rows (plan order, tokens
    shard_ranges(plan, world)[1][r]) of q, k, v, gates, dout. Data path:
      1. ssa_pool of the owned compression blocks (compression blocks nest in query blocks), summed
         over ranks (all-reduce, 2 x h_kv x n_cmp x d fp32 — 5 MB at C3);
      2. raw K/V all-gather on `comm_stream`, recorded in an event the forward waits on right before
         the selection / window branch, so the exchange overlaps the compression attention (a4/a5);
      3. forward and backward for the owned rows only (SSA_LOCAL_ROWS); dk, dv come back as fp32
         partials over every token (SSA_KV_GRAD_FP32) and are reduce-scattered to their owners.
    q_ranges: optional explicit query-block range of every rank of the group (hybrid_plan); default
    balanced by tokens. exchange="fetch" replaces step 2 by the one-sided fetch: the ranks exchange
    CUDA IPC handles of their K/V rows and the forward copies only the selection blocks its query blocks
    selected from their owners, after the compression attention and top-k (cfg.peers).
    Returns (out, dq, dk, dv, dgates) for the owned rows (dk, dv in k_loc's dtype)."""
    import dataclasses
    import torch
    from . import ssa
    if q_ranges is None:
        q_rng, tok = shard_ranges(plan, world)
    else:
        qo = plan.q_offsets_host()
        q_rng = [tuple(x) for x in q_ranges]
        tok = [(int(qo[a]), int(qo[b])) for a, b in q_rng]
    qb, qe = q_rng[rank]
    c2 = dataclasses.replace(cfg, flags=cfg.flags | ssa.SSA_INPUT_SORTED | ssa.SSA_KV_GRAD_FP32 | ssa.SSA_LOCAL_ROWS,
                             q_begin=qb, q_end=qe)
    dev = q_loc.device
    cur = torch.cuda.current_stream(dev)
    kc, vc = ssa.ssa_pool(plan, c2, k_loc, v_loc)
    all_reduce_sum(kc, group)
    all_reduce_sum(vc, group)
    if exchange == "fetch":
        import torch.distributed as dist
        k = torch.empty((plan.n,) + tuple(k_loc.shape[1:]), dtype=k_loc.dtype, device=dev)
        v = torch.empty_like(k)
        a, b = tok[rank]
        k[a:b] = k_loc
        v[a:b] = v_loc
        pk, pv, bases = exchange_peer_pointers(k_loc, v_loc, rank, world, group)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier(group=group)              # every rank's K/V rows are in place
        cf = dataclasses.replace(c2, kc_in=kc, vc_in=vc, peers=(pk, pv, [t[0] for t in tok] + [tok[-1][1]], rank))
        out, saved = ssa.ssa_forward(plan, cf, q_loc, k, v, gates_loc)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier(group=group)              # no rank frees rows another is still reading
        for base in bases:
            ssa.ipc_close(base)
    else:
        comm = comm_stream or torch.cuda.Stream(dev)
        comm.wait_stream(cur)                          # k_loc / v_loc are ready
        ev = torch.cuda.Event()
        with torch.cuda.stream(comm):
            k = torch.empty((plan.n,) + tuple(k_loc.shape[1:]), dtype=k_loc.dtype, device=dev)
            v = torch.empty_like(k)
            all_gather_rows(k, k_loc, tok, rank, group)
            all_gather_rows(v, v_loc, tok, rank, group)
            ev.record(comm)
        k.record_stream(cur)
        v.record_stream(cur)
        cf = dataclasses.replace(c2, kc_in=kc, vc_in=vc, kv_event=ev)
        out, saved = ssa.ssa_forward(plan, cf, q_loc, k, v, gates_loc)
    dq, dk, dv, dg = ssa.ssa_backward(plan, c2, saved, q_loc, k, v, gates_loc, dout_loc)
    dk_loc = reduce_scatter_rows(dk, tok, rank, group)
    dv_loc = reduce_scatter_rows(dv, tok, rank, group)
    return out, dq, dk_loc.to(k_loc.dtype), dv_loc.to(k_loc.dtype), dg


# ---------------------------------------------------------------------------------------------------
# Hybrid placement ("near-linear scaling to 8 needs hybrid splitting"). The query blocks of
# all shapes of the batch are laid end to end on one cost line (a query block of shape b costs
# ~ tokens(Q) * n_b: its rows against the n_b / m_cmp^3 compressed keys of its shape, the dominant
# compression branch) and the line is cut into `world` contiguous pieces of equal cost. A rank whose
# piece covers a shape entirely runs it whole (mode 1, no collective); a shape cut by one or more
# piece boundaries is sharded by query blocks (mode 2, ssa_step_sharded) over the contiguous sub-group
# of ranks that hold a piece of it, with unequal ranges.
# ---------------------------------------------------------------------------------------------------
def hybrid_plan(q_tokens, world: int):
    """q_tokens: per shape, the token counts of its query blocks (plan order). Returns one list per rank
    of (shape, q_begin, q_end, group) with group = the ascending tuple of ranks that share the shape
    (length 1: the shape runs whole on this rank). Deterministic: every rank computes the same plan."""
    import numpy as np
    n_tok = [int(np.sum(t)) for t in q_tokens]
    w = [np.asarray(t, np.float64) * n for t, n in zip(q_tokens, n_tok)]
    total = float(sum(x.sum() for x in w))
    out = [[] for _ in range(world)]
    if world <= 1 or total <= 0:
        out[0] = [(s, 0, len(t), (0,)) for s, t in enumerate(q_tokens)]
        return out
    pieces = {}          # shape -> {rank: [q_begin, q_end)}
    acc = 0.0
    for s, ws in enumerate(w):
        for Q, x in enumerate(ws):
            r = min(world - 1, int((acc + 0.5 * x) / total * world))   # rank of the block's cost midpoint
            acc += x
            rng = pieces.setdefault(s, {}).setdefault(r, [Q, Q + 1])
            rng[1] = Q + 1
        if not len(ws):
            pieces.setdefault(s, {})[min(world - 1, int(acc / total * world))] = [0, 0]
    for s in range(len(q_tokens)):
        grp = tuple(sorted(pieces[s]))
        for r in grp:
            a, b = pieces[s][r]
            out[r].append((s, a, b, grp))
    return out


def hybrid_makespan(q_tokens, plan):
    """Modelled cost (same model as hybrid_plan) of the busiest rank of a plan."""
    import numpy as np
    n_tok = [int(np.sum(t)) for t in q_tokens]
    return max((sum(float(np.sum(np.asarray(q_tokens[s][a:b], np.float64))) * n_tok[s] for s, a, b, _ in items)
                for items in plan), default=0.0)


class HybridBatch:
    """One rank's share of a batch of shapes under the hybrid placement (hybrid_plan):
    the shapes this rank holds entirely run as ONE batch plan (mode 1, no collective), the shapes cut by
    a piece boundary run ssa_step_sharded over their sub-group (mode 2). Every rank must construct it
    with the same arguments (it creates the sub-groups with dist.new_group in shape order).

    coords: list of host int32 [n_s, 4] arrays (batch index 0), one per shape; grid; ms = (m_cmp, m_slc,
    m_win, m_q); cfg: AttnCfg. step(tensors) with tensors[s] = (q, k, v, gates, dout) of shape s in its
    caller order returns {"whole": (shapes, out, dq, dk, dv, dgates) of the concatenated whole shapes or
    None, "split": {s: (plan-order rows [a, b), out, dq, dk, dv, dgates) of this rank's rows}}."""

    def __init__(self, coords, grid, ms, cfg, rank, world, device, exchange="allgather"):
        import numpy as np
        import torch
        import torch.distributed as dist
        from . import ssa
        self.ssa, self.cfg, self.rank, self.world, self.ms = ssa, cfg, rank, world, tuple(ms)
        self.grid = tuple(grid)
        self.exchange = exchange
        self.cdev = [torch.from_numpy(np.ascontiguousarray(c)).to(device) for c in coords]
        qt = [np.diff(ssa.ssa_build_blocks(cd, self.grid, 1, *self.ms).q_offsets_host()) for cd in self.cdev]
        self.plan = hybrid_plan(qt, world)
        self.groups, self.ranges = {}, {}
        for s in range(len(coords)):                   # every rank creates every sub-group, in shape order
            grp = next(g for items in self.plan for (ss, a, b, g) in items if ss == s)
            if len(grp) > 1:
                self.groups[s] = dist.new_group(list(grp)) if world > 1 else None
                self.ranges[s] = [next((a, b) for (ss, a, b, _) in self.plan[r] if ss == s) for r in grp]
        mine = self.plan[rank]
        self.whole = [s for (s, a, b, g) in mine if len(g) == 1]
        self.split = [(s, g) for (s, a, b, g) in mine if len(g) > 1]
        self.wcoords = None
        if self.whole:
            parts = []
            for i, s in enumerate(self.whole):
                c = np.array(coords[s], copy=True)
                c[:, 0] = i
                parts.append(c)
            self.wcoords = torch.from_numpy(np.concatenate(parts)).to(device)
        self.comm = torch.cuda.Stream(device)

    def step(self, tensors):
        import torch
        ssa = self.ssa
        res = {"whole": None, "split": {}}
        if self.whole:
            q, k, v, g, do = (torch.cat([tensors[s][i] for s in self.whole]) for i in range(5))
            plan = ssa.ssa_build_blocks(self.wcoords, self.grid, len(self.whole), *self.ms)
            out, saved = ssa.ssa_forward(plan, self.cfg, q, k, v, g)
            dq, dk, dv, dg = ssa.ssa_backward(plan, self.cfg, saved, q, k, v, g, do)
            res["whole"] = (list(self.whole), out, dq, dk, dv, dg)
        for s, grp in self.split:
            plan = ssa.ssa_build_blocks(self.cdev[s], self.grid, 1, *self.ms)
            qo = plan.q_offsets_host()
            a, b = self.ranges[s][grp.index(self.rank)]
            ta, tb = int(qo[a]), int(qo[b])
            rows = plan.perm()[ta:tb].long()
            loc = [x[rows] for x in tensors[s]]
            out = ssa_step_sharded(plan, self.cfg, *loc, rank=grp.index(self.rank), world=len(grp),
                                   group=self.groups[s], comm_stream=self.comm, q_ranges=self.ranges[s],
                                   exchange=self.exchange)
            res["split"][s] = ((ta, tb),) + tuple(out)
        return res
