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
