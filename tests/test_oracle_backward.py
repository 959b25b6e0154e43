"""Pins for oracle O9 (analytic backward): central finite differences of the oracle's own forward
(a different computation from the analytic chain rule), plus closed-form special cases
(SPEC.md:216-217)."""
import math

import numpy as np

from conftest import random_coords
import oracle as O

KW = dict(h_kv=2, T=2, m_cmp=2, m_slc=4, m_win=4, m_q=4)


def _problem(rng, n=30, G=8, batch=2, H=4, h_kv=2, d=3):
    c = random_coords(rng, n, G, batch)
    N = len(c)
    return (c, rng.standard_normal((N, H, d)), rng.standard_normal((N, h_kv, d)),
            rng.standard_normal((N, h_kv, d)), rng.uniform(0.1, 0.9, (N, H, 3)), rng.standard_normal((N, H, d)))


def test_finite_differences_all_inputs(rng):
    c, q, k, v, gates, dout = _problem(rng)
    f0 = O.ssa_forward(c, (8, 8, 8), 2, q, k, v, gates, **KW)
    I = f0.I                                   # hard routing: indices frozen (READING R15)
    dq, dk, dv, dg = O.ssa_backward(f0, q, k, v, gates, dout, h_kv=2)

    def loss(q_, k_, v_, g_):
        f = O.ssa_forward(c, (8, 8, 8), 2, q_, k_, v_, g_, I_override=I, plan=f0.plan, **KW)
        return float((f.out * dout).sum())

    h = 1e-5
    sel = np.random.Generator(np.random.PCG64(7))
    for name, arr, grad in (("q", q, dq), ("k", k, dk), ("v", v, dv), ("gates", gates, dg)):
        flat = arr.reshape(-1)
        gflat = grad.reshape(-1)
        for idx in sel.choice(flat.size, size=min(25, flat.size), replace=False):
            orig = flat[idx]
            flat[idx] = orig + h
            lp = loss(q, k, v, gates)
            flat[idx] = orig - h
            lm = loss(q, k, v, gates)
            flat[idx] = orig
            fd = (lp - lm) / (2 * h)
            assert abs(fd - gflat[idx]) <= 1e-5 * max(1.0, abs(fd)), (name, idx, fd, gflat[idx])


def test_zero_dout_and_single_token(rng):
    c, q, k, v, gates, dout = _problem(rng)
    f = O.ssa_forward(c, (8, 8, 8), 2, q, k, v, gates, **KW)
    for g in O.ssa_backward(f, q, k, v, gates, np.zeros_like(dout), h_kv=2):
        assert np.all(g == 0)
    # N = 1: softmax constant -> dq = dk = 0, dv = (sum_c w_c) dO summed over the group's heads
    c1 = np.array([[0, 1, 2, 3]])
    f = O.ssa_forward(c1, (8, 8, 8), 1, q[:1], k[:1], v[:1], gates[:1], **KW)
    dq, dk, dv, dg = O.ssa_backward(f, q[:1], k[:1], v[:1], gates[:1], dout[:1], h_kv=2)
    assert np.allclose(dq, 0, atol=1e-15) and np.allclose(dk, 0, atol=1e-15)
    w = gates[0].sum(axis=1)
    want = np.stack([(w[2 * g:2 * g + 2, None] * dout[0, 2 * g:2 * g + 2]).sum(axis=0) for g in range(2)])
    assert np.allclose(dv[0], want, atol=1e-14)


def test_gradient_sparsity(rng):
    """A token that is in no selected block, whose window holds only itself... gets k/v gradient only
    through its own window and the compression pool: here we check that with gates
    (0, 1, 0) a token outside every selected block gets exactly zero dk/dv."""
    c, q, k, v, gates, dout = _problem(rng, n=60)
    g010 = np.broadcast_to([0.0, 1.0, 0.0], gates.shape).copy()
    kw = dict(KW, T=1)
    f = O.ssa_forward(c, (8, 8, 8), 2, q, k, v, g010, **kw)
    _, dk, dv, _ = O.ssa_backward(f, q, k, v, g010, dout, h_kv=2)
    plan = f.plan
    C = plan.offsets["slc"]
    for g in range(2):
        used = set()
        for b in f.I[:, g].reshape(-1):
            if b >= 0:
                used.update(plan.perm[C[b]:C[b + 1]].tolist())
        for t in range(len(c)):
            if t not in used:
                assert np.all(dk[t, g] == 0) and np.all(dv[t, g] == 0)


def test_block_kv_grad_equals_full_backward(rng):
    """The per-block gradient functions used for full-size parity (block_kv_grad = raw_kv_grad_block +
    compression_kv_grad pool share) equal ssa_backward's dk / dv on every selection block of a ragged
    two-item problem (so they inherit its finite-difference pins); chunking and threads do not matter."""
    c, q, k, v, gates, dout = _problem(rng, n=90, H=6, d=4)
    kw = dict(KW, T=3)
    f = O.ssa_forward(c, (8, 8, 8), 2, q, k, v, gates, **kw)
    dq, dk, dv, dg = O.ssa_backward(f, q, k, v, gates, dout, h_kv=2)
    plan = f.plan
    P = plan.perm
    scale = 1.0 / math.sqrt(q.shape[2])
    C = plan.offsets["slc"]
    res = O.block_kv_grad(plan, q[P], k[P], v[P], f.k_cmp, f.v_cmp, gates[P], dout[P], f.I, 2, scale,
                          range(plan.n_blocks("slc")), workers=3)
    for B, (gk, gv) in res.items():
        assert np.allclose(gk, dk[P][C[B]:C[B + 1]], rtol=0, atol=1e-12)
        assert np.allclose(gv, dv[P][C[B]:C[B + 1]], rtol=0, atol=1e-12)
    b = 1
    c0, c1 = int(plan.batch_blocks["cmp"][b]), int(plan.batch_blocks["cmp"][b + 1])
    cols = np.arange(c0, c1)
    a = O.compression_kv_grad(plan, q[P], f.k_cmp, f.v_cmp, gates[P], dout[P], 2, scale, b, cols, chunk=5)
    z = O.compression_kv_grad(plan, q[P], f.k_cmp, f.v_cmp, gates[P], dout[P], 2, scale, b, cols, chunk=10 ** 6)
    assert np.allclose(a[0], z[0], rtol=0, atol=1e-12) and np.allclose(a[1], z[1], rtol=0, atol=1e-12)


def test_shifted_window_ssa(rng):
    """Shifted-window SSA (reading R20): shift 0 is plain SSA; with shift 2 the output differs only in
    the window term (cmp / slc branches unchanged) and the analytic gradients match central finite
    differences of the shifted forward (indices frozen)."""
    c, q, k, v, gates, dout = _problem(rng)
    f0 = O.ssa_forward(c, (8, 8, 8), 2, q, k, v, gates, **KW)
    fs0 = O.ssa_forward_shifted(c, (8, 8, 8), 2, q, k, v, gates, shift=0, **KW)
    assert np.allclose(fs0.out, f0.out, rtol=0, atol=1e-14)
    g_plain = O.ssa_backward(f0, q, k, v, gates, dout, h_kv=2)
    g_s0 = O.ssa_backward_shifted(fs0, c, q, k, v, gates, dout, shift=0, m_win=4, h_kv=2)
    for a, b in zip(g_plain, g_s0):
        assert np.allclose(a, b, rtol=0, atol=1e-12)
    fs = O.ssa_forward_shifted(c, (8, 8, 8), 2, q, k, v, gates, shift=2, **KW)
    assert np.allclose(fs.o["cmp"], f0.o["cmp"]) and np.allclose(fs.o["slc"], f0.o["slc"])
    assert not np.allclose(fs.o["win"], f0.o["win"])
    grads = O.ssa_backward_shifted(fs, c, q, k, v, gates, dout, shift=2, m_win=4, h_kv=2)

    def loss():
        f = O.ssa_forward_shifted(c, (8, 8, 8), 2, q, k, v, gates, shift=2, I_override=fs.I, **KW)
        return float((f.out * dout).sum())

    h = 1e-5
    sel = np.random.Generator(np.random.PCG64(9))
    for arr, grad in zip((q, k, v, gates), grads):
        flat, gflat = arr.reshape(-1), grad.reshape(-1)
        for idx in sel.choice(flat.size, size=10, replace=False):
            orig = flat[idx]
            flat[idx] = orig + h
            lp = loss()
            flat[idx] = orig - h
            lm = loss()
            flat[idx] = orig
            fd = (lp - lm) / (2 * h)
            assert abs(fd - gflat[idx]) <= 1e-5 * max(1.0, abs(fd))
