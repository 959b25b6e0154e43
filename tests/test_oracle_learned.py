"""Pins for the oracle's learned compression delta (Eq. 7, READING R17) and gate projection (Eq. 6 /
P:153, READING R18): reductions to the pinned mean pool, closed forms, a coordinate-driven loop,
a pure-python sigmoid, and central finite differences of the whole learned backward."""
import math

import numpy as np

from conftest import random_coords
import oracle as O

KW = dict(h_kv=2, T=2, m_cmp=2, m_slc=4, m_win=4, m_q=4)


def test_identity_kernel_is_mean_pool(rng):
    """W[loc] = I, b = 0: the learned delta is exactly the mean pool (R4), with and without PE."""
    c = random_coords(rng, 120, 8, 2)
    plan = O.block_build(c, (8, 8, 8), 2, 2, 4, 4, 4)
    x = rng.standard_normal((len(c), 2, 5))
    pe = rng.standard_normal((8, 2, 5))
    W = np.broadcast_to(np.eye(5), (8, 2, 5, 5)).copy()
    for p in (None, pe):
        assert np.allclose(O.compress_learned(plan, x, W, None, p), O.compress(plan, x, p), rtol=0, atol=1e-14)


def test_zero_kernel_bias_and_singletons(rng):
    """W = 0: every block is b. A one-token block is W[loc] (x + PE[loc]) + b (no averaging)."""
    c = random_coords(rng, 80, 8, 1)
    plan = O.block_build(c, (8, 8, 8), 1, 2, 4, 4, 4)
    x = rng.standard_normal((len(c), 2, 3))
    b = rng.standard_normal((2, 4))
    out = O.compress_learned(plan, x, np.zeros((8, 2, 4, 3)), b)
    assert np.allclose(out, np.broadcast_to(b, out.shape), rtol=0, atol=0)
    W = rng.standard_normal((8, 2, 4, 3))
    pe = rng.standard_normal((8, 2, 3))
    out = O.compress_learned(plan, x, W, b, pe)
    C = plan.offsets["cmp"]
    n_single = 0
    for j in range(len(C) - 1):
        if C[j + 1] - C[j] == 1:
            t = int(C[j])
            sx, sy, sz = (int(v) % 2 for v in plan.sorted_coords[t, 1:])
            loc = (sx * 2 + sy) * 2 + sz
            for g in range(2):
                assert np.allclose(out[j, g], W[loc, g] @ (x[t, g] + pe[loc, g]) + b[g], rtol=0, atol=1e-13)
            n_single += 1
    assert n_single >= 3


def test_coordinate_loop(rng):
    """Blocks and local offsets taken from the coordinates (pure python), one math.fsum per output."""
    m = 2
    c = random_coords(rng, 150, 8, 2)
    plan = O.block_build(c, (8, 8, 8), 2, m, 4, 4, 4)
    N = len(c)
    x = rng.standard_normal((N, 2, 3))              # ORIGINAL order here
    W = rng.standard_normal((m ** 3, 2, 4, 3))
    b = rng.standard_normal((2, 4))
    pe = rng.standard_normal((m ** 3, 2, 3))
    out = O.compress_learned(plan, x[plan.perm], W, b, pe)
    groups = {}
    for i, (bb, xx, yy, zz) in enumerate(c.tolist()):
        groups.setdefault((bb, xx // m, yy // m, zz // m), []).append((i, ((xx % m) * m + yy % m) * m + zz % m))
    for j, key in enumerate(map(tuple, plan.block_coords["cmp"].tolist())):
        toks = groups[key]
        for g in range(2):
            for e in range(4):
                want = math.fsum(W[l, g, e, f] * (x[i, g, f] + pe[l, g, f]) for i, l in toks for f in range(3)) / len(toks)
                assert abs(out[j, g, e] - (want + b[g, e])) < 1e-12


def test_gate_projection_closed_forms(rng):
    x = rng.standard_normal((7, 6))
    g0 = O.gate_projection(x, np.zeros((6, 12)), np.zeros(12), 4)
    assert g0.shape == (7, 4, 3) and np.all(g0 == 0.5)
    Wg, bg = rng.standard_normal((6, 12)), rng.standard_normal(12)
    g = O.gate_projection(x, Wg, bg, 4)
    for t in range(7):
        for h in range(4):
            for c in range(3):
                z = math.fsum(x[t, f] * Wg[f, h * 3 + c] for f in range(6)) + bg[h * 3 + c]
                assert abs(g[t, h, c] - 1.0 / (1.0 + math.exp(-z))) < 1e-15


def test_identity_learned_equals_plain_ssa(rng):
    """Identity kernels + gates taken from the projection reproduce ssa_forward / ssa_backward."""
    c = random_coords(rng, 40, 8, 2)
    N, H, h_kv, d, C = len(c), 4, 2, 3, 5
    q, k, v = rng.standard_normal((N, H, d)), rng.standard_normal((N, h_kv, d)), rng.standard_normal((N, h_kv, d))
    x, Wg, bg = rng.standard_normal((N, C)), rng.standard_normal((C, 3 * H)), rng.standard_normal(3 * H)
    dout = rng.standard_normal((N, H, d))
    eye = (np.broadcast_to(np.eye(d), (8, h_kv, d, d)).copy(), np.zeros((h_kv, d)))
    fl, gates = O.ssa_forward_learned(c, (8, 8, 8), 2, q, k, v, x, conv_k=eye, conv_v=eye, gate=(Wg, bg), **KW)
    f = O.ssa_forward(c, (8, 8, 8), 2, q, k, v, gates, **KW)
    assert np.array_equal(fl.I, f.I) and np.allclose(fl.out, f.out, rtol=0, atol=1e-13)
    gl = O.ssa_backward_learned(fl, q, k, v, x, gates, dout, conv_k=eye, conv_v=eye, gate=(Wg, bg), h_kv=h_kv)
    g = O.ssa_backward(f, q, k, v, gates, dout, h_kv=h_kv)
    for a, b in zip(gl[:3], g[:3]):
        assert np.allclose(a, b, rtol=0, atol=1e-12)


def test_learned_finite_differences(rng):
    """Central differences (h = 1e-5) of sum(out * dO) w.r.t. every input of the learned forward, with the
    selection indices frozen (R15): q, k, v, x, W_k, b_k, W_v, b_v, W_g, b_g."""
    c = random_coords(rng, 30, 8, 2)
    N, H, h_kv, d, C = len(c), 4, 2, 3, 4
    q, k, v = rng.standard_normal((N, H, d)), rng.standard_normal((N, h_kv, d)), rng.standard_normal((N, h_kv, d))
    x = rng.standard_normal((N, C))
    Wk, bk = rng.standard_normal((8, h_kv, d, d)), rng.standard_normal((h_kv, d))
    Wv, bv = rng.standard_normal((8, h_kv, d, d)), rng.standard_normal((h_kv, d))
    Wg, bg = rng.standard_normal((C, 3 * H)), rng.standard_normal(3 * H)
    dout = rng.standard_normal((N, H, d))
    f0, gates = O.ssa_forward_learned(c, (8, 8, 8), 2, q, k, v, x, conv_k=(Wk, bk), conv_v=(Wv, bv), gate=(Wg, bg), **KW)
    grads = O.ssa_backward_learned(f0, q, k, v, x, gates, dout, conv_k=(Wk, bk), conv_v=(Wv, bv), gate=(Wg, bg), h_kv=h_kv)

    def loss():
        f, _ = O.ssa_forward_learned(c, (8, 8, 8), 2, q, k, v, x, conv_k=(Wk, bk), conv_v=(Wv, bv), gate=(Wg, bg),
                                     I_override=f0.I, **KW)
        return float((f.out * dout).sum())

    h = 1e-5
    sel = np.random.Generator(np.random.PCG64(5))
    for name, arr, grad in zip(("q", "k", "v", "x", "Wk", "bk", "Wv", "bv", "Wg", "bg"),
                               (q, k, v, x, Wk, bk, Wv, bv, Wg, bg), grads):
        flat, gflat = arr.reshape(-1), np.asarray(grad).reshape(-1)
        for idx in sel.choice(flat.size, size=min(12, flat.size), replace=False):
            orig = flat[idx]
            flat[idx] = orig + h
            lp = loss()
            flat[idx] = orig - h
            lm = loss()
            flat[idx] = orig
            fd = (lp - lm) / (2 * h)
            assert abs(fd - gflat[idx]) <= 1e-5 * max(1.0, abs(fd)), (name, idx, fd, gflat[idx])
