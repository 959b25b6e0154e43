"""Pins for oracle O2-O8 (compression, attention branches, Eq. 8 scores, top-k, gates).

The reference values come from outside the oracle: SPEC worked examples (tests/golden), closed forms,
a pure-Python brute-force attention (math.exp loops, written here, not the oracle's numpy routine),
special cases in which SSA reduces to full attention, and invariants.
"""
import json
import math
import os

import numpy as np
import pytest

from conftest import random_coords
import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def brute_attention(q, k, v, scale):
    """Pure-python Eq. 4-5 for one query row list against key/value row lists."""
    out, lses = [], []
    for qi in q:
        s = [scale * math.fsum(a * b for a, b in zip(qi, kj)) for kj in k]
        mx = max(s)
        p = [math.exp(x - mx) for x in s]
        den = math.fsum(p)
        out.append([math.fsum(p[j] * v[j][c] for j in range(len(v))) / den for c in range(len(v[0]))])
        lses.append(mx + math.log(den))
    return np.array(out), np.array(lses)


def test_dense_spec_example():
    ex = json.load(open(os.path.join(GOLD, "dense_attention_spec_example.json")))
    o, lse, p = O.dense_attention(np.array(ex["q"]), np.array(ex["k"]), np.array(ex["v"]), ex["scale"])
    assert abs(o[0, 0] - ex["expected_o"]) < 1e-15
    assert abs(o[0, 0] - math.e / (1 + math.e)) < 1e-15
    assert abs(lse[0] - math.log(1 + math.e)) < 1e-15
    assert abs(p.sum() - 1) < 1e-15


def test_dense_special_cases(rng):
    # single token -> its value, lse = scale q.k
    q, k, v = rng.standard_normal((1, 8)), rng.standard_normal((1, 8)), rng.standard_normal((1, 5))
    o, lse, _ = O.dense_attention(q, k, v, 0.3)
    assert np.allclose(o, v, atol=1e-15) and abs(lse[0] - 0.3 * float((q @ k.T)[0, 0])) < 1e-14
    # identical keys -> mean of values
    k = np.repeat(rng.standard_normal((1, 8)), 7, axis=0)
    v = rng.standard_normal((7, 3))
    o, _, _ = O.dense_attention(rng.standard_normal((4, 8)), k, v, 0.5)
    assert np.allclose(o, v.mean(axis=0)[None], atol=1e-14)
    # random vs pure-python brute force; adversarial logits do not overflow
    q, k, v = rng.standard_normal((5, 6)) * 9, rng.standard_normal((11, 6)) * 9, rng.standard_normal((11, 4))
    o, lse, p = O.dense_attention(q, k, v, 1.0)
    ob, lb = brute_attention(q.tolist(), k.tolist(), v.tolist(), 1.0)
    assert np.allclose(o, ob, rtol=0, atol=1e-12) and np.allclose(lse, lb, rtol=1e-14, atol=1e-12)
    # convex hull
    assert np.all(o <= v.max(axis=0) + 1e-12) and np.all(o >= v.min(axis=0) - 1e-12)


def test_pool_spec_example():
    ex = json.load(open(os.path.join(GOLD, "scores_topk_gate_spec_examples.json")))
    c = np.array([[0, 0, 0, 0], [0, 1, 0, 0]])
    plan = O.block_build(c, (4, 4, 4), 1, 4, 4, 4, 4)
    x = np.array(ex["pool_tokens"])[:, None, :]
    assert np.allclose(O.compress(plan, x)[0, 0], ex["pool_expected"], atol=0)
    # singleton blocks -> identity
    plan1 = O.block_build(c, (4, 4, 4), 1, 1, 1, 1, 1)
    assert np.array_equal(O.compress(plan1, x), x)


def test_scores_and_topk_spec_examples():
    ex = json.load(open(os.path.join(GOLD, "scores_topk_gate_spec_examples.json")))
    # 2 tokens? No: one query token with h_s = 2 rows, two cmp blocks in one slc block.
    c = np.array([[0, 0, 0, 0], [0, 4, 0, 0]])          # two cmp blocks (m=4) in one slc block (m=8)
    plan = O.block_build(c, (8, 8, 8), 1, 4, 8, 8, 8)
    probs = {(0, 0): np.array(ex["scores_probs_rows_by_cmp"])}     # rows (h_s=2) x cmp blocks
    sc = O.block_scores(plan, probs, 1)[(0, 0)]
    assert sc.shape == (1,) and abs(sc[0] - ex["scores_expected"]) < 1e-15
    assert O.topk_select(np.array(ex["topk_scores"]), ex["topk_T"]).tolist() == ex["topk_expected"]
    # T >= N -> all, ascending, padded
    assert O.topk_select(np.array([0.1, 0.9, 0.5]), 5).tolist() == [0, 1, 2, -1, -1]


def test_topk_against_lexsort(rng):
    for _ in range(50):
        n = int(rng.integers(1, 40))
        s = rng.integers(0, 6, size=n).astype(float) / 5      # many exact ties
        T = int(rng.integers(1, 10))
        got = O.topk_select(s, T)
        order = np.lexsort((np.arange(n), -s))               # independent library ranking
        want = sorted(order[:min(T, n)].tolist())
        assert got[:len(want)].tolist() == want and np.all(got[len(want):] == -1)
        sel = got[got >= 0]
        uns = np.setdiff1d(np.arange(n), sel)
        if len(uns):
            assert s[sel].min() >= s[uns].max()              # selection optimality


def test_gate_examples(rng):
    ex = json.load(open(os.path.join(GOLD, "scores_topk_gate_spec_examples.json")))
    X = rng.standard_normal((3, 2, 4))
    g = np.broadcast_to(np.array(ex["gate"]), (3, 2, 3))
    assert np.allclose(O.gate_combine(X, X, X, g), ex["gate_factor_expected"] * X, atol=1e-15)
    A, B, C = rng.standard_normal((3, 3, 2, 4))
    assert np.array_equal(O.gate_combine(A, B, C, np.broadcast_to([1.0, 0, 0], (3, 2, 3))), A)


def _small_problem(rng, n=60, G=8, batch=1, h_kv=2, h_s=2, d=4):
    c = random_coords(rng, n, G, batch)
    N = len(c)
    q = rng.standard_normal((N, h_kv * h_s, d))
    k = rng.standard_normal((N, h_kv, d))
    v = rng.standard_normal((N, h_kv, d))
    gates = rng.uniform(0.05, 0.95, (N, h_kv * h_s, 3))
    return c, q, k, v, gates


def _full_attention_bruteforce(c, q, k, v, h_kv, scale):
    """Pure-python full attention per batch item (the reduction target)."""
    N, H, d = q.shape
    h_s = H // h_kv
    out = np.zeros((N, H, v.shape[2]))
    for b in np.unique(c[:, 0]):
        idx = np.nonzero(c[:, 0] == b)[0]
        for h in range(H):
            g = h // h_s
            o, _ = brute_attention(q[idx, h].tolist(), k[idx, g].tolist(), v[idx, g].tolist(), scale)
            out[idx, h] = o
    return out


def test_reductions_to_full_attention(rng):
    c, q, k, v, gates = _small_problem(rng, n=40, G=8, batch=2)
    h_kv, d = 2, 4
    scale = 1 / math.sqrt(d)
    full = _full_attention_bruteforce(c, q, k, v, h_kv, scale)
    N = len(c)
    # selection branch with T >= N_slc -> full attention
    f = O.ssa_forward(c, (8, 8, 8), 2, q, k, v, gates, h_kv=h_kv, T=64, m_cmp=2, m_slc=4, m_win=4, m_q=4)
    assert np.allclose(f.o["slc"], full, atol=1e-12)
    # window branch with m_win >= G -> full attention (O7)
    f = O.ssa_forward(c, (8, 8, 8), 2, q, k, v, gates, h_kv=h_kv, T=2, m_cmp=2, m_slc=4, m_win=8, m_q=4)
    assert np.allclose(f.o["win"], full, atol=1e-12)
    # compression with m_cmp = 1 (no PE) -> per-token full attention (O3)
    f = O.ssa_forward(c, (8, 8, 8), 2, q, k, v, gates, h_kv=h_kv, T=2, m_cmp=1, m_slc=4, m_win=4, m_q=4)
    assert np.allclose(f.o["cmp"], full, atol=1e-12)
    # whole SSA with gates (0,1,0) and T >= N_slc -> full attention
    g010 = np.broadcast_to([0.0, 1.0, 0.0], gates.shape)
    f = O.ssa_forward(c, (8, 8, 8), 2, q, k, v, g010, h_kv=h_kv, T=64, m_cmp=2, m_slc=4, m_win=4, m_q=4)
    assert np.allclose(f.out, full, atol=1e-12)
    # N = 1 -> (sum of gates) * v
    c1 = np.array([[0, 3, 2, 1]])
    f = O.ssa_forward(c1, (8, 8, 8), 1, q[:1], k[:1], v[:1], gates[:1], h_kv=h_kv, T=4, m_cmp=2, m_slc=4,
                      m_win=4, m_q=4)
    want = gates[0].sum(axis=1)[:, None] * np.repeat(v[0], 2, axis=0)
    assert np.allclose(f.out[0], want, atol=1e-15)


def test_alg1_tile_independence_and_equivalence(rng):
    c, q, k, v, gates = _small_problem(rng, n=70, G=8)
    h_kv = 2
    f = O.ssa_forward(c, (8, 8, 8), 1, q, k, v, gates, h_kv=h_kv, T=3, m_cmp=2, m_slc=4, m_win=4, m_q=2)
    plan = f.plan
    P = plan.perm
    ref = None
    for B_k in (1, 2, 7, 64):                                   # SPEC.md:378 / acceptance 2
        o, l = O.selection_attention_alg1(plan, q[P], k[P], v[P], f.I, h_kv, 0.5, B_k=B_k)
        if ref is None:
            ref = (o, l)
        assert np.allclose(o, ref[0], atol=1e-12) and np.allclose(l, ref[1], atol=1e-12)
    o2, l2 = O.selection_attention(plan, q[P], k[P], v[P], f.I, h_kv, 0.5)
    assert np.allclose(ref[0], o2, atol=1e-12) and np.allclose(ref[1], l2, atol=1e-12)
    # Alg. 1 at m_q = 1 against brute force over the selected tokens for a few tokens
    f1 = O.ssa_forward(c, (8, 8, 8), 1, q, k, v, gates, h_kv=h_kv, T=2, m_cmp=2, m_slc=4, m_win=4, m_q=1)
    o1, l1 = O.selection_attention_alg1(f1.plan, q[f1.plan.perm], k[f1.plan.perm], v[f1.plan.perm], f1.I,
                                        h_kv, 0.5, B_k=3)
    C = f1.plan.offsets["slc"]
    for t in (0, 13, 42):
        for g in range(h_kv):
            toks = np.concatenate([np.arange(C[b], C[b + 1]) for b in f1.I[t, g] if b >= 0])
            kk = k[f1.plan.perm][toks, g].tolist()
            vv = v[f1.plan.perm][toks, g].tolist()
            ob, lb = brute_attention(q[f1.plan.perm][t, 2 * g:2 * g + 2].tolist(), kk, vv, 0.5)
            assert np.allclose(o1[t, 2 * g:2 * g + 2], ob, atol=1e-12)
            assert np.allclose(l1[t, 2 * g:2 * g + 2], lb, atol=1e-12)


def test_probability_rows_and_score_checksum(rng):
    c, q, k, v, gates = _small_problem(rng, n=80, G=8, batch=2)
    f = O.ssa_forward(c, (8, 8, 8), 2, q, k, v, gates, h_kv=2, T=2, m_cmp=2, m_slc=4, m_win=4, m_q=4)
    plan = f.plan
    _, _, probs = O.compression_attention(plan, q[plan.perm], f.k_cmp, f.v_cmp, 2, 0.5)
    for p in probs.values():
        assert np.allclose(p.sum(axis=1), 1.0, atol=1e-14)          # softmax rows sum to 1
    Cq = plan.offsets["q"]
    for (Q, g), sc in f.scores.items():
        assert abs(sc.sum() - (Cq[Q + 1] - Cq[Q]) * 2) < 1e-12       # Σ_B score = |Q| * h_s
    # single slc block covering everything -> score = |Q| * h_s
    f = O.ssa_forward(c, (8, 8, 8), 2, q, k, v, gates, h_kv=2, T=1, m_cmp=2, m_slc=8, m_win=4, m_q=4)
    for (Q, g), sc in f.scores.items():
        assert sc.shape == (1,) and abs(sc[0] - (f.plan.offsets["q"][Q + 1] - f.plan.offsets["q"][Q]) * 2) < 1e-12


def test_token_order_invariance(rng):
    c, q, k, v, gates = _small_problem(rng, n=60, G=8, batch=2)
    kw = dict(h_kv=2, T=2, m_cmp=2, m_slc=4, m_win=4, m_q=4)
    f1 = O.ssa_forward(c, (8, 8, 8), 2, q, k, v, gates, **kw)
    sh = rng.permutation(len(c))
    f2 = O.ssa_forward(c[sh], (8, 8, 8), 2, q[sh], k[sh], v[sh], gates[sh], **kw)
    assert np.allclose(f1.out[sh], f2.out, atol=1e-12)
    assert np.array_equal(f1.I, f2.I)


def test_window_locality(rng):
    c, q, k, v, gates = _small_problem(rng, n=60, G=8)
    kw = dict(h_kv=2, T=2, m_cmp=2, m_slc=4, m_win=4, m_q=4)
    f1 = O.ssa_forward(c, (8, 8, 8), 1, q, k, v, gates, **kw)
    t = 5
    w = tuple(c[t, 1:] // 4)
    outside = np.array([tuple(r[1:] // 4) != w for r in c])
    k2, v2, q2 = k.copy(), v.copy(), q.copy()
    k2[outside] = 0
    v2[outside] = 0
    q2[outside] = 0
    f2 = O.ssa_forward(c, (8, 8, 8), 1, q2, k2, v2, gates, **kw)
    assert np.allclose(f1.o["win"][t], f2.o["win"][t], atol=1e-14)


def _blocks_from_coords(coords, m):
    """Pure-python grouping of token indices by (b, x//m, y//m, z//m) — independent of block_build."""
    groups = {}
    for i, (b, x, y, z) in enumerate(np.asarray(coords).tolist()):
        groups.setdefault((b, x // m, y // m, z // m), []).append(i)
    return groups


def test_eq8_triple_loop_multi_block(rng):
    """Eq. 8 as a pure-python triple loop — sum over t in Q, over the h_s shared heads and
    over the compression blocks whose coordinates lie inside each selection block — on inputs with 8
    selection blocks of 2^3 compression blocks each ("random case -> naive triple loop").
    Everything is derived from the coordinates here: the pooled keys (mean per compression cell), the
    probabilities (math.exp softmax per (t, head)) and the containment cmp -> slc (bx_c // 2 == bx_s);
    a compression block credited to the wrong selection block, a dropped head or a dropped token fails."""
    m_cmp, m_slc, m_q, h_kv, h_s, d = 2, 4, 4, 2, 3, 5
    c = random_coords(rng, 300, 8, 2)
    N = len(c)
    q = rng.standard_normal((N, h_kv * h_s, d))
    k = rng.standard_normal((N, h_kv, d))
    scale = 1.0 / math.sqrt(d)
    plan = O.block_build(c, (8, 8, 8), 2, m_cmp, m_slc, m_slc, m_q)
    P = plan.perm
    k_cmp = O.compress(plan, k[P])
    _, _, probs = O.compression_attention(plan, q[P], k_cmp, k_cmp, h_kv, scale)
    scores = O.block_scores(plan, probs, h_kv)
    cmp_groups = _blocks_from_coords(c, m_cmp)
    slc_groups = _blocks_from_coords(c, m_slc)
    q_groups = _blocks_from_coords(c, m_q)
    ratio = m_slc // m_cmp
    n_checked = 0
    for qkey, qtoks in q_groups.items():
        b = qkey[0]
        ckeys = sorted(kk for kk in cmp_groups if kk[0] == b)
        skeys = sorted(kk for kk in slc_groups if kk[0] == b)
        for g in range(h_kv):
            kbar = {kk: [math.fsum(k[i][g][e] for i in cmp_groups[kk]) / len(cmp_groups[kk]) for e in range(d)]
                    for kk in ckeys}
            want = {sk: 0.0 for sk in skeys}
            for t in qtoks:                                            # sum over t in Q
                for s in range(h_s):                                   # sum over the shared heads
                    h = g * h_s + s
                    logit = {kk: scale * math.fsum(q[t][h][e] * kbar[kk][e] for e in range(d)) for kk in ckeys}
                    mx = max(logit.values())
                    den = math.fsum(math.exp(x - mx) for x in logit.values())
                    for kk in ckeys:                                   # sum over cmp blocks in the slc block
                        sk = (b, kk[1] // ratio, kk[2] // ratio, kk[3] // ratio)
                        want[sk] += math.exp(logit[kk] - mx) / den
            # oracle's query block / selection block numbering: sorted block coordinates of the plan
            Q = int(plan.tok_block["q"][plan.inv_perm[qtoks[0]]])
            s0 = int(plan.batch_blocks["slc"][b])
            got = scores[(Q, g)]
            assert len(got) == len(skeys) >= 3
            for j, sk in enumerate(skeys):
                assert tuple(plan.block_coords["slc"][s0 + j]) == sk
                assert abs(got[j] - want[sk]) <= 1e-12 * max(1.0, want[sk])
            n_checked += 1
    assert n_checked >= 8
    assert max(len([kk for kk in cmp_groups if (kk[0], kk[1] // 2, kk[2] // 2, kk[3] // 2) == sk])
               for sk in slc_groups) >= 4                              # several cmp blocks per slc block


def test_compress_pe_pins(rng):
    """Eq. 7 with the intra-block PE: with k = 0, k^cmp of a block is the mean
    of the PE rows at the local offsets (x % m, y % m, z % m) of its ACTIVE tokens; with k != 0 it is the
    naive per-block mean of k_j + PE[local(j)] (PE added before pooling). Grouping and local offsets are
    computed here from the coordinates."""
    m, h_kv, d = 4, 2, 3
    c = random_coords(rng, 200, 16, 2)
    N = len(c)
    pe = rng.standard_normal((m ** 3, h_kv, d))
    plan = O.block_build(c, (16, 16, 16), 2, m, 2 * m, 2 * m, 2 * m)
    groups = _blocks_from_coords(c, m)
    kc0 = O.compress(plan, np.zeros((N, h_kv, d)), pe)
    k = rng.standard_normal((N, h_kv, d))
    kc1 = O.compress(plan, k[plan.perm], pe)
    for j, bc in enumerate(plan.block_coords["cmp"].tolist()):
        toks = groups[tuple(bc)]
        loc = [((c[i][1] % m) * m + c[i][2] % m) * m + c[i][3] % m for i in toks]
        want0 = np.mean([pe[l] for l in loc], axis=0)
        want1 = np.mean([k[i] + pe[l] for i, l in zip(toks, loc)], axis=0)
        assert np.allclose(kc0[j], want0, rtol=0, atol=1e-14)
        assert np.allclose(kc1[j], want1, rtol=0, atol=1e-14)
    # a PE that depends only on z % m: swapping the x and y offsets of the table changes nothing,
    # swapping x and z does (the table is indexed (x*m + y)*m + z)
    pz = np.zeros((m, m, m, h_kv, d))
    pz[:, :, 1] = 1.0
    a = O.compress(plan, np.zeros((N, h_kv, d)), pz.reshape(m ** 3, h_kv, d))
    b = O.compress(plan, np.zeros((N, h_kv, d)), np.swapaxes(pz, 0, 1).reshape(m ** 3, h_kv, d))
    cz = O.compress(plan, np.zeros((N, h_kv, d)), np.swapaxes(pz, 0, 2).reshape(m ** 3, h_kv, d))
    assert np.array_equal(a, b) and not np.array_equal(a, cz)
