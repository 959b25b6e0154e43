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
