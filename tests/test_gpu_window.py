"""Sparse 3D (shifted-)window attention (the SS-VAE's attention layer; SSA's window branch on
its own) through ssa.window_attention, against an independent reference built from the pinned
oracle dense attention (oracle.dense_attention / dense_attention_backward) applied window by window.
Windows: floor((x + s) / m_win) per batch item, s = 0 (aligned) or m_win / 2 (shifted)."""
import math

import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import record, to_dev
from paper_2505_17412_b200 import ssa
from ssa_workload import batch_coords, make_inputs, sphere_shell

pytestmark = pytest.mark.gpu


def _reference(coords, q, k, v, dout, h_kv, m, shift):
    N, H, d = q.shape
    h_s = H // h_kv
    scale = 1.0 / math.sqrt(d)
    key = np.concatenate([coords[:, :1], (coords[:, 1:] + shift) // m], axis=1)
    _, win = np.unique(key, axis=0, return_inverse=True)
    out, dq, dk, dv = (np.zeros_like(x) for x in (q, q, k, v))
    for w in np.unique(win):
        t = np.nonzero(win.ravel() == w)[0]
        for g in range(h_kv):
            for s in range(h_s):
                h = g * h_s + s
                o, _, p = O.dense_attention(q[t, h], k[t, g], v[t, g], scale)
                out[t, h] = o
                gq, gk, gv = O.dense_attention_backward(q[t, h], k[t, g], v[t, g], p, o, dout[t, h], scale)
                dq[t, h] += gq
                dk[t, g] += gk
                dv[t, g] += gv
    return out, dq, dk, dv


@pytest.mark.parametrize("window_only", [True, False])
@pytest.mark.parametrize("shift", [0, 4])
def test_window_attention(shift, window_only):
    coords = batch_coords([sphere_shell(24, 9.0, 2.0), sphere_shell(24, 7.0, 2.0)])
    grid = (24, 24, 24)
    inp = make_inputs(coords, grid, 2, 8, 2, 64, "bf16", seed=11)
    q, k, v, do = (to_dev(x, torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.dout))
    out, ctx = ssa.window_attention(torch.from_numpy(coords).cuda(), grid, 2, 8, q, k, v, h_kv=2, shift=shift,
                                    window_only=window_only)
    assert ctx[2].used_tcgen05
    dq, dk, dv = ssa.window_attention_backward(ctx, q, k, v, do)
    torch.cuda.synchronize()
    ref = _reference(coords, inp.q, inp.k, inp.v, inp.dout, 2, 8, shift)
    test = f"test_window_attention[shift={shift},window_only={window_only}]"
    errs = {n: record(test, n, x.float().cpu().numpy().astype(np.float64), r, 2e-2, stored_bf16=True)
            for n, x, r in zip(("out", "dq", "dk", "dv"), (out, dq, dk, dv), ref)}
    assert all(e <= 2e-2 for e in errs.values()), errs


def test_window_covering_grid_is_full_attention():
    """m_win >= grid: one window per batch item, i.e. full attention over the item."""
    coords = batch_coords([sphere_shell(16, 6.0, 2.0)])
    grid = (16, 16, 16)
    inp = make_inputs(coords, grid, 1, 8, 2, 64, "bf16", seed=12)
    q, k, v = (to_dev(x, torch.bfloat16) for x in (inp.q, inp.k, inp.v))
    out, ctx = ssa.window_attention(torch.from_numpy(coords).cuda(), grid, 1, 16, q, k, v, h_kv=2)
    torch.cuda.synchronize()
    N, H, d = inp.q.shape
    ref = np.zeros_like(inp.q)
    for h in range(H):
        ref[:, h] = O.dense_attention(inp.q[:, h], inp.k[:, h // 4], inp.v[:, h // 4], 1.0 / math.sqrt(d))[0]
    assert record("test_window_covering_grid_is_full_attention", "out", out.float().cpu().numpy().astype(np.float64),
                  ref, 2e-2, stored_bf16=True) <= 2e-2


def test_window_only_skips_branches_and_matches_composition():
    """SSA_WINDOW_ONLY launches neither the compression kernel nor the compressed-key backward, and gives
    the same window-branch result as the full step with gates (0, 0, 1) (same kernels, same order)."""
    coords = batch_coords([sphere_shell(32, 13.0, 2.0)])
    grid = (32, 32, 32)
    inp = make_inputs(coords, grid, 1, 16, 2, 64, "bf16", seed=14)
    q, k, v, do = (to_dev(x, torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.dout))
    c = torch.from_numpy(coords).cuda()
    res = {}
    for wo in (False, True):
        ssa.profile_reset()
        ssa.profile_enable(True)
        out, ctx = ssa.window_attention(c, grid, 1, 8, q, k, v, h_kv=2, window_only=wo)
        grads = ssa.window_attention_backward(ctx, q, k, v, do)
        torch.cuda.synchronize()
        ssa.profile_enable(False)
        res[wo] = (out,) + tuple(grads), {n: ssa.profile_read(n)[1] for n in ("tc_cmp_fwd", "tc_bwd_cmp_kv")}
    assert res[False][1] == {"tc_cmp_fwd": 1, "tc_bwd_cmp_kv": 1}
    assert res[True][1] == {"tc_cmp_fwd": 0, "tc_bwd_cmp_kv": 0}
    for a, b in zip(res[True][0], res[False][0]):
        # GPU vs GPU (same kernels; the window-only run may differ by one bf16 ulp where a skipped
        # branch's exact zero changes an fp32 rounding): |a - b| <= 2^-8 |b| element-wise
        a, b = a.float(), b.float()
        assert torch.equal(a, b) or bool(((a - b).abs() <= 2.0 ** -8 * b.abs()).all())


@pytest.mark.parametrize("shift", [0, 4])
def test_shifted_window_ssa(shift):
    """SSA with shifted windows (reading R20): ssa.shifted_window_ssa = SSA_NO_WINDOW on
    the plan of the coordinates + SSA_WINDOW_ONLY | SSA_ACCUMULATE on the plan of the shifted ones,
    against oracle.ssa_forward_shifted / ssa_backward_shifted (GPU indices fed to the oracle). shift 0
    must also reproduce the plain step."""
    coords = batch_coords([sphere_shell(32, 13.0, 2.0), sphere_shell(32, 9.0, 2.0)])
    grid = (32, 32, 32)
    inp = make_inputs(coords, grid, 2, 16, 2, 64, "bf16", seed=15)
    q, k, v, g, do = (to_dev(x, torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout))
    cfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=4, dtype=torch.bfloat16)
    c = torch.from_numpy(coords).cuda()
    out, ctx = ssa.shifted_window_ssa(c, grid, 2, 4, 8, shift, cfg, q, k, v, g)
    dq, dk, dv, dg = ssa.shifted_window_ssa_backward(ctx, q, k, v, g, do)
    torch.cuda.synchronize()
    I = ctx[4].indices().cpu().numpy().astype(np.int64)
    kw = dict(h_kv=2, T=4, m_cmp=4, m_slc=8, m_win=8, m_q=8)
    f = O.ssa_forward_shifted(coords, grid, 2, inp.q, inp.k, inp.v, inp.gates, shift=shift, I_override=I, **kw)
    ref = O.ssa_backward_shifted(f, coords, inp.q, inp.k, inp.v, inp.gates, inp.dout, shift=shift, m_win=8, h_kv=2)
    test = f"test_shifted_window_ssa[{shift}]"
    errs = {n: record(test, n, x.float().cpu().numpy().astype(np.float64), r, 2e-2, stored_bf16=True)
            for n, x, r in zip(("out", "dq", "dk", "dv", "dgates"), (out, dq, dk, dv, dg), (f.out,) + tuple(ref))}
    assert all(e <= 2e-2 for e in errs.values()), errs
