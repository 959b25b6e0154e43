"""GPU parity of the learned compression delta (Eq. 7, reading R17) and the fused gate projection
(Eq. 6 / P:153, reading R18), forward and backward, against oracle.ssa_forward_learned /
ssa_backward_learned on the same seeded inputs (GPU indices fed to the oracle):
out, dq, dk, dv, dx and the weight gradients dW_k, db_k, dW_v, db_v, dW_g, db_g, undiscounted."""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import record, to_dev, topk_end_to_end_check

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2}


def _params(rng, m3, h_kv, d, C, H):
    Wk = (np.eye(d)[None, None] + 0.25 * rng.standard_normal((m3, h_kv, d, d)) / np.sqrt(d)).astype(np.float32)
    Wv = (np.eye(d)[None, None] + 0.25 * rng.standard_normal((m3, h_kv, d, d)) / np.sqrt(d)).astype(np.float32)
    bk, bv = (0.1 * rng.standard_normal((2, h_kv, d))).astype(np.float32)
    Wg = (rng.standard_normal((C, 3 * H)) / np.sqrt(C)).astype(np.float32)
    bg = (0.5 * rng.standard_normal(3 * H)).astype(np.float32)
    return Wk, bk, Wv, bv, Wg, bg


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_learned_delta_and_gate_projection(dtype):
    from paper_2505_17412_b200 import ssa
    from ssa_workload import batch_coords, make_inputs, round_to_bf16, sphere_shell
    rng = np.random.Generator(np.random.PCG64(31))
    coords = batch_coords([sphere_shell(24, 9.0, 2.0), sphere_shell(24, 7.0, 2.0)])
    grid, batch, H, h_kv, d, C = (24, 24, 24), 2, 8, 2, 64, 96
    inp = make_inputs(coords, grid, batch, H, h_kv, d, dtype, seed=8)
    x = rng.standard_normal((len(coords), C)).astype(np.float32)
    if dtype == "bf16":
        x = round_to_bf16(x)
    Wk, bk, Wv, bv, Wg, bg = _params(rng, 64, h_kv, d, C, H)
    kw = dict(h_kv=h_kv, T=4, m_cmp=4, m_slc=8, m_win=8, m_q=8)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    dev = torch.device("cuda")
    f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev, torch.float32)
    learned = ssa.Learned(conv_k_w=f32(Wk), conv_k_b=f32(bk), conv_v_w=f32(Wv), conv_v_b=f32(bv),
                          x=to_dev(x, tdt), gate_w=f32(Wg), gate_b=f32(bg))
    plan = ssa.ssa_build_blocks(torch.from_numpy(coords).to(dev), grid, batch, 4, 8, 8, 8)
    cfg = ssa.AttnCfg(h_q=H, h_kv=h_kv, d=d, top_k=4, dtype=tdt, learned=learned, flags=ssa.SSA_SAVE_SCORES)
    q, k, v, do = (to_dev(a, tdt) for a in (inp.q, inp.k, inp.v, inp.dout))
    out, saved = ssa.ssa_forward(plan, cfg, q, k, v, None)
    dq, dk, dv, dg = ssa.ssa_backward(plan, cfg, saved, q, k, v, None, do)
    torch.cuda.synchronize()
    assert saved.used_tcgen05 == (dtype == "bf16")
    I = saved.indices().cpu().numpy().astype(np.int64)
    conv = dict(conv_k=(Wk, bk), conv_v=(Wv, bv), gate=(Wg, bg))
    f_free, _ = O.ssa_forward_learned(coords, grid, batch, inp.q, inp.k, inp.v, x, **conv, **kw)
    mism, amb = topk_end_to_end_check(f_free.plan, f_free.scores, I, 4, 1e-4 if dtype == "bf16" else 1e-6)
    assert mism == 0, (mism, amb)
    f, gates = O.ssa_forward_learned(coords, grid, batch, inp.q, inp.k, inp.v, x, I_override=I, **conv, **kw)
    ref = O.ssa_backward_learned(f, inp.q, inp.k, inp.v, x, gates, inp.dout, h_kv=h_kv, **conv)
    g = learned.grads
    got = dict(out=out, dq=dq, dk=dk, dv=dv, dx=g["dx"], d_conv_k_w=g["d_conv_k_w"], d_conv_k_b=g["d_conv_k_b"],
               d_conv_v_w=g["d_conv_v_w"], d_conv_v_b=g["d_conv_v_b"], d_gate_w=g["d_gate_w"], d_gate_b=g["d_gate_b"])
    want = dict(out=f.out, dq=ref[0], dk=ref[1], dv=ref[2], dx=ref[3], d_conv_k_w=ref[4], d_conv_k_b=ref[5],
                d_conv_v_w=ref[6], d_conv_v_b=ref[7], d_gate_w=ref[8], d_gate_b=ref[9])
    kc, vc = saved.k_cmp()
    got["k_cmp"] = kc.permute(1, 0, 2)
    want["k_cmp"] = f.k_cmp
    test = f"test_learned_delta_and_gate_projection[{dtype}]"
    b16 = {"out", "dq", "dk", "dv", "dx"} if dtype == "bf16" else set()   # stored in the input dtype
    errs = {n: record(test, n, got[n].float().cpu().numpy().astype(np.float64), want[n], TOL[dtype], stored_bf16=n in b16)
            for n in got}
    bad = {n: e for n, e in errs.items() if e > TOL[dtype]}
    assert not bad, (bad, errs)


def test_identity_learned_equals_mean_pool():
    """Identity kernels, zero biases and the gate projection's own gates fed as inputs: the learned path
    reproduces the plain path (same kernels downstream of the pool) to fp32 rounding of the pool."""
    from paper_2505_17412_b200 import ssa
    from ssa_workload import batch_coords, make_inputs, sphere_shell
    coords = batch_coords([sphere_shell(32, 13.0, 2.0)])
    inp = make_inputs(coords, (32, 32, 32), 1, 16, 2, 64, "bf16", seed=9)
    dev = torch.device("cuda")
    eye = torch.eye(64, device=dev).expand(64, 2, 64, 64).contiguous()
    zero = torch.zeros(2, 64, device=dev)
    plan = ssa.ssa_build_blocks(torch.from_numpy(coords).to(dev), (32, 32, 32), 1, 4, 8, 8, 8)
    q, k, v, g, do = (to_dev(a, torch.bfloat16) for a in (inp.q, inp.k, inp.v, inp.gates, inp.dout))
    base = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=4, dtype=torch.bfloat16)
    o0, s0 = ssa.ssa_forward(plan, base, q, k, v, g)
    r0 = ssa.ssa_backward(plan, base, s0, q, k, v, g, do)
    lcfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=4, dtype=torch.bfloat16,
                       learned=ssa.Learned(conv_k_w=eye, conv_k_b=zero, conv_v_w=eye, conv_v_b=zero))
    o1, s1 = ssa.ssa_forward(plan, lcfg, q, k, v, g)
    r1 = ssa.ssa_backward(plan, lcfg, s1, q, k, v, g, do)
    torch.cuda.synchronize()
    assert torch.equal(s0.indices(), s1.indices())
    for a, b in zip((o0,) + tuple(r0), (o1,) + tuple(r1)):
        a, b = a.float(), b.float()
        assert bool(((a - b).abs() <= 2.0 ** -7 * b.abs() + 1e-3 * b.pow(2).mean().sqrt()).all())
