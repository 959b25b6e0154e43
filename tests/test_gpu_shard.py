"""Query-block sharding (SURVEY §8e mode 2) on one GPU with virtual ranks: the shards' collectives
are replaced by concatenation / summation. Rows a shard owns must equal the unsharded run bit for bit
(same kernels, same per-row work); dK / dV partial sums may differ only by fp32 summation order."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("force_simt", [False, True])
def test_virtual_ranks(force_simt):
    import torch
    from paper_2505_17412_b200 import ssa
    from paper_2505_17412_b200.shard import balanced_q_ranges
    from ssa_workload import config_coords, make_inputs
    c, grid, batch = config_coords("C2")
    inp = make_inputs(c, grid, batch, 16, 2, 64, "bf16", seed=11)
    dev = torch.device("cuda")
    plan = ssa.ssa_build_blocks(torch.from_numpy(c).to(dev), grid, batch, 4, 8, 8, 8)
    perm = plan.perm().cpu().numpy()
    flags = ssa.SSA_INPUT_SORTED | (ssa.SSA_FORCE_SIMT if force_simt else 0)
    t = [torch.from_numpy(x[perm]).to(dev, dtype=torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)]
    cfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=8, dtype=torch.bfloat16, flags=flags)
    out0, saved0 = ssa.ssa_forward(plan, cfg, *t[:4])
    g0 = [x.clone() for x in ssa.ssa_backward(plan, cfg, saved0, *t)]
    out0 = out0.clone()
    qo = plan.offsets(ssa.LEVEL_Q).cpu().numpy()
    ranges = balanced_q_ranges(qo, 3)
    assert ranges[0][0] == 0 and ranges[-1][1] == len(qo) - 1
    out = torch.zeros_like(out0)
    dq = torch.zeros_like(g0[0])
    dk = torch.zeros(g0[1].shape, dtype=torch.float32, device=dev)
    dv = torch.zeros_like(dk)
    for qb, qe in ranges:
        cr = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=8, dtype=torch.bfloat16, flags=flags | ssa.SSA_KV_GRAD_FP32,
                         q_begin=qb, q_end=qe)
        o, sv = ssa.ssa_forward(plan, cr, *t[:4])
        gq, gk, gv, gg = ssa.ssa_backward(plan, cr, sv, *t)
        a, b = int(qo[qb]), int(qo[qe])
        out[a:b] = o[a:b]
        dq[a:b] = gq[a:b]
        dk += gk.float()
        dv += gv.float()
        assert torch.equal(gg[a:b], g0[3][a:b])
    assert torch.equal(out, out0)
    assert torch.equal(dq, g0[0])
    for got, ref in ((dk, g0[1].float()), (dv, g0[2].float())):
        # fp32 partials summed vs the unsharded bf16 output: the reference's own rounding (2^-8) plus
        # fp32 summation-order differences
        err = ((got - ref).abs() - 2.0 ** -8 * ref.abs()).clamp_min(0).max().item() / ref.pow(2).mean().sqrt().item()
        assert err < 1e-3, err


def _c2_sorted(seed=11):
    import torch
    from paper_2505_17412_b200 import ssa
    from ssa_workload import config_coords, make_inputs
    c, grid, batch = config_coords("C2")
    inp = make_inputs(c, grid, batch, 16, 2, 64, "bf16", seed=seed)
    dev = torch.device("cuda")
    plan = ssa.ssa_build_blocks(torch.from_numpy(c).to(dev), grid, batch, 4, 8, 8, 8)
    perm = plan.perm().cpu().numpy()
    t = [torch.from_numpy(x[perm]).to(dev, dtype=torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)]
    return plan, t


def test_local_rows_pool_and_kv_event():
    """Mode-2 data path on one GPU with virtual ranks, exactly as ssa_step_sharded drives it but with the
    collectives replaced by sums / concatenation: ssa_pool of each rank's own rows (SSA_LOCAL_ROWS), the
    pooled keys summed over ranks and passed as kc_in / vc_in, the raw K/V produced on a side stream and
    signalled through kv_event, forward + backward on local row tensors. Owned rows of out / dq / dgates
    are bit-identical to the unsharded run; the summed dk / dv partials match it up to fp32 order."""
    import dataclasses
    import torch
    from paper_2505_17412_b200 import ssa
    from paper_2505_17412_b200.shard import shard_ranges
    plan, (q, k, v, g, do) = _c2_sorted()
    base = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=8, dtype=torch.bfloat16, flags=ssa.SSA_INPUT_SORTED)
    out0, saved0 = ssa.ssa_forward(plan, base, q, k, v, g)
    ref = [x.clone() for x in ssa.ssa_backward(plan, base, saved0, q, k, v, g, do)]
    out0 = out0.clone()
    q_rng, tok = shard_ranges(plan, 3)
    flags = base.flags | ssa.SSA_KV_GRAD_FP32 | ssa.SSA_LOCAL_ROWS
    cfgs = [dataclasses.replace(base, flags=flags, q_begin=a, q_end=b) for a, b in q_rng]
    kc = torch.zeros(2, plan.n_blocks[ssa.LEVEL_CMP], 64, device="cuda")
    vc = torch.zeros_like(kc)
    for cr, (a, b) in zip(cfgs, tok):
        pk, pv = ssa.ssa_pool(plan, cr, k[a:b].contiguous(), v[a:b].contiguous())
        kc += pk
        vc += pv
    kc0, vc0 = saved0.k_cmp()
    assert torch.equal(kc, kc0) and torch.equal(vc, vc0)          # same summation order as the full pool
    dk = torch.zeros(k.shape, dtype=torch.float32, device="cuda")
    dv = torch.zeros_like(dk)
    side = torch.cuda.Stream()
    for cr, (a, b) in zip(cfgs, tok):
        ev = torch.cuda.Event()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):                              # "all-gather" of K/V on a side stream
            kk, vv = k.clone(), v.clone()
            ev.record(side)
        kk.record_stream(torch.cuda.current_stream())
        vv.record_stream(torch.cuda.current_stream())
        cf = dataclasses.replace(cr, kc_in=kc, vc_in=vc, kv_event=ev)
        o, sv = ssa.ssa_forward(plan, cf, q[a:b].contiguous(), kk, vv, g[a:b].contiguous())
        gq, gk, gv, gg = ssa.ssa_backward(plan, cr, sv, q[a:b].contiguous(), kk, vv, g[a:b].contiguous(),
                                          do[a:b].contiguous())
        assert torch.equal(o, out0[a:b]) and torch.equal(gq, ref[0][a:b]) and torch.equal(gg, ref[3][a:b])
        dk += gk
        dv += gv
    for got, want in ((dk, ref[1].float()), (dv, ref[2].float())):
        err = ((got - want).abs() - 2.0 ** -8 * want.abs()).clamp_min(0).max().item() / want.pow(2).mean().sqrt().item()
        assert err < 1e-3, err


def _proc(rank, world, port, path, exchange="allgather"):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_17412_b200.shard import shard_ranges, ssa_step_sharded
    from paper_2505_17412_b200 import ssa
    plan, (q, k, v, g, do) = _c2_sorted()
    cfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=8, dtype=torch.bfloat16)
    _, tok = shard_ranges(plan, world)
    a, b = tok[rank]
    loc = [x[a:b].contiguous() for x in (q, k, v, g, do)]
    res = ssa_step_sharded(plan, cfg, *loc, rank=rank, world=world, exchange=exchange)
    torch.cuda.synchronize()
    torch.save([x.cpu() for x in res] + [torch.tensor([a, b])], f"{path}/r{rank}.pt")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["allgather", "fetch"])
def test_two_process_sharded_step(tmp_path, exchange):
    """ssa_step_sharded end to end in two processes (gloo on one GPU; the driver's boxes have one GPU):
    per-rank inputs (own rows of q, k, v, gates, dO only), pooled-key all-reduce, K/V all-gather on a side
    stream overlapping the compression branch (or, exchange="fetch", the one-sided fetch of only the
    selected blocks through CUDA IPC peer mappings), dK/dV reduce-scatter. Each rank's out / dq / dgates equal
    the unsharded run's rows bit for bit; its dk / dv rows match up to fp32 summation order."""
    import socket
    import torch
    import torch.multiprocessing as mp
    from paper_2505_17412_b200 import ssa
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=_proc, args=(r, 2, port, str(tmp_path), exchange)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=600)
        assert p.exitcode == 0
    plan, (q, k, v, g, do) = _c2_sorted()
    base = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=8, dtype=torch.bfloat16, flags=ssa.SSA_INPUT_SORTED)
    out0, saved0 = ssa.ssa_forward(plan, base, q, k, v, g)
    ref = ssa.ssa_backward(plan, base, saved0, q, k, v, g, do)
    torch.cuda.synchronize()
    covered = 0
    for r in range(2):
        o, dq, dk, dv, dg, ab = torch.load(f"{tmp_path}/r{r}.pt")
        a, b = ab.tolist()
        covered += b - a
        assert torch.equal(o, out0[a:b].cpu()) and torch.equal(dq, ref[0][a:b].cpu()) and torch.equal(dg, ref[3][a:b].cpu())
        for got, want in ((dk, ref[1][a:b].cpu()), (dv, ref[2][a:b].cpu())):
            got, want = got.float(), want.float()
            # both sides rounded to bf16 from fp32 sums taken in different orders: one bf16 ulp
            assert bool(((got - want).abs() <= 2.0 ** -7 * want.abs() + 1e-4 * want.pow(2).mean().sqrt()).all())
    assert covered == plan.n


def _hybrid_shapes():
    from ssa_workload import batch_coords, sphere_shell
    return [batch_coords([sphere_shell(32, r, 2.0)]) for r in (9.0, 12.0, 14.0)]


def _hybrid_proc(rank, world, port, path, exchange):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_17412_b200 import ssa
    from paper_2505_17412_b200.shard import HybridBatch
    from ssa_workload import make_inputs
    shapes = _hybrid_shapes()
    tens = []
    for s, c in enumerate(shapes):
        inp = make_inputs(c, (32, 32, 32), 1, 16, 2, 64, "bf16", seed=40 + s)
        tens.append([torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)])
    cfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=4, dtype=torch.bfloat16)
    hb = HybridBatch(shapes, (32, 32, 32), (4, 8, 8, 8), cfg, rank, world, torch.device("cuda"), exchange=exchange)
    res = hb.step(tens)
    torch.cuda.synchronize()
    w = res["whole"]
    save = {"whole": None if w is None else (w[0],) + tuple(x.cpu() for x in w[1:]),
            "split": {s: (v[0],) + tuple(x.cpu() for x in v[1:]) for s, v in res["split"].items()},
            "plan": hb.plan}
    torch.save(save, f"{path}/h{rank}.pt")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["allgather", "fetch"])
def test_two_process_hybrid_batch(tmp_path, exchange):
    """Hybrid placement of a 3-shape batch on 2 ranks (shard.HybridBatch, the C4 bench path
    at N > 1): the cost-line cut splits the middle shape over both ranks (mode 2) while the others run
    whole (mode 1). Every shape's out / dq / dgates equal a single-GPU run of that shape (whole shapes:
    the batch plan computes each item independently; split shape: owned rows bit for bit); dk / dv
    within one bf16 ulp (fp32 partial sums in another order)."""
    import socket
    import torch
    import torch.multiprocessing as mp
    from paper_2505_17412_b200 import ssa
    from ssa_workload import make_inputs
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=_hybrid_proc, args=(r, 2, port, str(tmp_path), exchange)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=600)
        assert p.exitcode == 0
    res = [torch.load(f"{tmp_path}/h{r}.pt") for r in range(2)]
    assert any(len(g) > 1 for items in res[0]["plan"] for (_, _, _, g) in items), "expected a split shape"
    cfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=4, dtype=torch.bfloat16)
    shapes = _hybrid_shapes()
    ref = []
    for s, c in enumerate(shapes):
        inp = make_inputs(c, (32, 32, 32), 1, 16, 2, 64, "bf16", seed=40 + s)
        t = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)]
        plan = ssa.ssa_build_blocks(torch.from_numpy(c).cuda(), (32, 32, 32), 1, 4, 8, 8, 8)
        o, sv = ssa.ssa_forward(plan, cfg, *t[:4])
        g = ssa.ssa_backward(plan, cfg, sv, *t)
        torch.cuda.synchronize()
        ref.append((plan.perm().cpu().long(), o.cpu(), *(x.cpu() for x in g)))

    def close(a, b):
        a, b = a.float(), b.float()
        return bool(((a - b).abs() <= 2.0 ** -7 * b.abs() + 1e-4 * b.pow(2).mean().sqrt()).all())

    seen = {s: 0 for s in range(len(shapes))}
    for r in range(2):
        w = res[r]["whole"]
        if w is not None:
            off = 0
            for s in w[0]:
                n = len(shapes[s])
                for got, want in zip(w[1:], ref[s][1:]):
                    assert close(got[off:off + n], want)
                off += n
                seen[s] += n
        for s, (ab, out, dq, dk, dv, dg) in res[r]["split"].items():
            perm = ref[s][0][ab[0]:ab[1]]
            assert torch.equal(out, ref[s][1][perm]) and torch.equal(dq, ref[s][2][perm]) and torch.equal(dg, ref[s][5][perm])
            assert close(dk, ref[s][3][perm]) and close(dv, ref[s][4][perm])
            seen[s] += ab[1] - ab[0]
    assert all(seen[s] == len(shapes[s]) for s in seen)
