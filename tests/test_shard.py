"""Multi-process host logic of the N>1 path on CPU (gloo, world size 2): shape assignment is a
disjoint cover, LPT balances the C4 batch, and the max-over-ranks timing reduction works."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2505_17412_b200.shard import lpt_assign, rank_items


def test_lpt_cover_and_balance():
    from ssa_workload import CONFIGS, sphere_shell
    n = [sphere_shell(*s).shape[0] for s in CONFIGS["C4"]["shapes"]]
    for world in (1, 2, 4, 8):
        parts = lpt_assign([x * x for x in n], world)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(n)))
        loads = [sum(n[i] ** 2 for i in p) for p in parts]
        # LPT bound: makespan <= 4/3 OPT (and OPT >= max item, total/world)
        assert max(loads) <= 4 / 3 * max(max(x * x for x in n), sum(x * x for x in n) / world) + 1e-6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_17412_b200.shard import max_over_ranks, rank_items
    items = rank_items([100, 300, 200, 50], rank, world)
    m = max_over_ranks(10.0 + rank)
    q.put((rank, items, m))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][2] == 11.0 and res[1][2] == 11.0
    items = sorted(res[0][1] + res[1][1])
    assert items == [0, 1, 2, 3]
    assert res[0][1] == rank_items([100, 300, 200, 50], 0, 2)


def test_balanced_q_ranges_cover():
    from paper_2505_17412_b200.shard import balanced_q_ranges
    import numpy as np
    rng = np.random.Generator(np.random.PCG64(3))
    sizes = rng.integers(1, 200, size=500)
    off = np.concatenate([[0], np.cumsum(sizes)])
    for world in (1, 2, 3, 8):
        r = balanced_q_ranges(off, world)
        assert r[0][0] == 0 and r[-1][1] == 500
        assert all(a <= b for a, b in r) and all(r[i][1] == r[i + 1][0] for i in range(world - 1))
        loads = [off[b] - off[a] for a, b in r]
        assert max(loads) <= off[-1] / world + sizes.max()


def _coll_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_17412_b200.shard import all_gather_rows, all_reduce_sum, reduce_scatter_rows
    tok = [(0, 5), (5, 12)]                             # uneven ranges (padded exchange)
    full = torch.arange(12 * 3, dtype=torch.float32).view(12, 3) * (rank + 1)
    a, b = tok[rank]
    g = all_gather_rows(torch.zeros(12, 3), full[a:b], tok, rank)
    rs = reduce_scatter_rows(full, tok, rank)
    s = all_reduce_sum(torch.full((4,), float(rank + 1)))
    q.put((rank, g.tolist(), rs.tolist(), s.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_collectives_uneven_ranges():
    """Mode-2 exchange helpers on gloo, world size 2, uneven token ranges: all-gather of the owned rows
    rebuilds the full tensor from each rank's own rows, reduce-scatter gives each rank the sum over ranks
    of its own rows, all-reduce sums."""
    import torch
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_coll_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict((r, (g, rs, s)) for r, g, rs, s in (q.get(timeout=120) for _ in ps))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    base = torch.arange(36, dtype=torch.float32).view(12, 3)
    want_g = torch.cat([base[:5] * 1, base[5:] * 2])
    for r in (0, 1):
        assert torch.equal(torch.tensor(res[r][0]), want_g)
        assert res[r][2] == [3.0] * 4
    assert torch.equal(torch.tensor(res[0][1]), base[:5] * 3)
    assert torch.equal(torch.tensor(res[1][1]), base[5:] * 3)


def _c4_q_tokens():
    import numpy as np
    from ssa_workload import CONFIGS, sphere_shell
    out = []
    for sh in CONFIGS["C4"]["shapes"]:
        c = sphere_shell(*sh)
        out.append(np.unique(c // 8, axis=0, return_counts=True)[1])   # tokens per 8^3 query block
    return out


def test_hybrid_plan_cover_and_balance():
    """Hybrid placement of the C4 batch: every query block of every shape is owned by exactly
    one rank; a shape's sub-group is the contiguous set of ranks holding a piece of it and every member
    agrees on it; the modelled makespan is within 2% of total / world at 1, 2, 4, 8 ranks (plain LPT of
    whole shapes: 0.35 at 8 ranks)."""
    from paper_2505_17412_b200.shard import hybrid_makespan, hybrid_plan
    qt = _c4_q_tokens()
    total = sum(float(t.sum()) ** 2 for t in qt)
    for world in (1, 2, 3, 4, 8):
        plan = hybrid_plan(qt, world)
        assert len(plan) == world
        for s, t in enumerate(qt):
            pieces = sorted((a, b, r, g) for r, items in enumerate(plan) for (ss, a, b, g) in items if ss == s)
            assert pieces[0][0] == 0 and pieces[-1][1] == len(t)
            assert all(pieces[i][1] == pieces[i + 1][0] for i in range(len(pieces) - 1))
            grp = tuple(sorted(p[2] for p in pieces))
            assert all(p[3] == grp for p in pieces) and grp == tuple(range(grp[0], grp[-1] + 1))
        assert total / world / hybrid_makespan(qt, plan) >= 0.98
    lpt = lpt_assign([float(t.sum()) ** 2 for t in qt], 8)
    assert total / 8 / max(sum(float(qt[i].sum()) ** 2 for i in p) for p in lpt) < 0.4
