"""Full-size GPU parity (BASELINE configs C3 and C4 at their real token counts, in the launch
configuration bench.py times): outputs and dq are checked against the float64 oracle for a sample of
query blocks the oracle can compute one by one (largest, smallest and random blocks); dk / dv, which
depend on every row of a batch item, are checked through exact identities that hold at any size:

  sum_t dv[t, g] = sum over rows (t, s) of group g of (w_cmp + w_slc + w_win) * dO[t, (g, s)]
      (every branch's attention rows sum to 1, and the mean-pool backward preserves the sum)
  sum_t dk[t, g] = 0
      (sum_j dS_rj = sum_j P_rj (dP_rj - D_r) = 0 for every row r and branch)
"""
import math

import numpy as np
import pytest

import oracle as O
from gpu_util import rel_err, run_gpu

pytestmark = pytest.mark.gpu


def _sample_blocks(plan_o, n_random, rng):
    Cq = plan_o.offsets["q"]
    sizes = np.diff(Cq)
    pick = {int(np.argmax(sizes)), int(np.argmin(sizes))}
    pick |= set(int(x) for x in rng.choice(len(sizes), size=min(n_random, len(sizes)), replace=False))
    return sorted(pick)


def _check_blocks(inp, kw, r, plan_o, blocks):
    """Oracle forward + dq for the rows of the sampled query blocks (GPU indices for selection)."""
    N, H, d = inp.q.shape
    h_kv = kw["h_kv"]
    h_s = H // h_kv
    scale = 1.0 / math.sqrt(d)
    P = plan_o.perm
    qs = inp.q[P].astype(np.float64)
    ks = inp.k[P].astype(np.float64)
    vs = inp.v[P].astype(np.float64)
    gs = inp.gates[P].astype(np.float64)
    dos = inp.dout[P].astype(np.float64)
    k_cmp, v_cmp = O.compress(plan_o, ks), O.compress(plan_o, vs)
    Cq, Cs, Cw = plan_o.offsets["q"], plan_o.offsets["slc"], plan_o.offsets["win"]
    out_g = r["out"][P]
    dq_g = r["dq"][P]
    dg_g = r["dgates"][P]
    errs = {"out": [], "dq": [], "dgates": []}
    refs = {"out": [], "dq": [], "dgates": []}
    gots = {"out": [], "dq": [], "dgates": []}
    n_amb = 0
    for Q in blocks:
        a, b_ = int(Cq[Q]), int(Cq[Q + 1])
        bi = int(plan_o.sorted_coords[a, 0])
        c0, c1 = int(plan_o.batch_blocks["cmp"][bi]), int(plan_o.batch_blocks["cmp"][bi + 1])
        s0, s1 = int(plan_o.batch_blocks["slc"][bi]), int(plan_o.batch_blocks["slc"][bi + 1])
        w = int(plan_o.tok_block["win"][a])
        for g in range(h_kv):
            rows = qs[a:b_, g * h_s:(g + 1) * h_s].reshape(-1, d)
            drow = dos[a:b_, g * h_s:(g + 1) * h_s].reshape(-1, d)
            wt = gs[a:b_, g * h_s:(g + 1) * h_s].reshape(-1, 3)
            oc, _, pc = O.dense_attention(rows, k_cmp[c0:c1, g], v_cmp[c0:c1, g], scale)
            per = pc.sum(axis=0)
            sc = np.zeros(s1 - s0)
            np.add.at(sc, plan_o.cmp_to_slc[c0:c1] - s0, per)
            want = O.topk_select(sc, kw["T"], base=s0)
            got = r["I"][Q, g]
            if not np.array_equal(want, got):
                srt = np.sort(sc)[::-1]
                T = kw["T"]
                assert len(srt) > T and (srt[T - 1] - srt[T]) / srt[T - 1] < 1e-4, (Q, g, want, got)
                n_amb += 1
            kt = np.concatenate([np.arange(Cs[x], Cs[x + 1]) for x in got if x >= 0])
            os_, _, ps = O.dense_attention(rows, ks[kt, g], vs[kt, g], scale)
            wa, wb = int(Cw[w]), int(Cw[w + 1])
            ow, _, pw = O.dense_attention(rows, ks[wa:wb, g], vs[wa:wb, g], scale)
            outr = wt[:, 0:1] * oc + wt[:, 1:2] * os_ + wt[:, 2:3] * ow
            dgr = np.stack([(drow * o).sum(axis=1) for o in (oc, os_, ow)], axis=1)
            dqr = np.zeros_like(rows)
            for i, (kk, vv, pp, oo) in enumerate(((k_cmp[c0:c1, g], v_cmp[c0:c1, g], pc, oc),
                                                  (ks[kt, g], vs[kt, g], ps, os_),
                                                  (ks[wa:wb, g], vs[wa:wb, g], pw, ow))):
                dqi, _, _ = O.dense_attention_backward(rows, kk, vv, pp, oo, wt[:, i:i + 1] * drow, scale)
                dqr += dqi
            for name, ref, gpu in (("out", outr, out_g[a:b_, g * h_s:(g + 1) * h_s].reshape(-1, d)),
                                   ("dq", dqr, dq_g[a:b_, g * h_s:(g + 1) * h_s].reshape(-1, d)),
                                   ("dgates", dgr, dg_g[a:b_, g * h_s:(g + 1) * h_s].reshape(-1, 3))):
                refs[name].append(ref)
                gots[name].append(gpu)
    u = 2.0 ** -8
    for name in refs:
        errs[name] = rel_err(np.concatenate(gots[name]), np.concatenate(refs[name]), u)
    return errs, n_amb


def _identities(inp, r, h_kv):
    N, H, d = inp.q.shape
    h_s = H // h_kv
    w = inp.gates.astype(np.float64).sum(axis=2)                       # [N, H]
    wdo = w[..., None] * inp.dout.astype(np.float64)                     # [N, H, d]
    res = {}
    for g in range(h_kv):
        want_v = wdo[:, g * h_s:(g + 1) * h_s].sum(axis=(0, 1))
        got_v = r["dv"][:, g].sum(axis=0)
        res[f"sum_dv_g{g}"] = float(np.max(np.abs(got_v - want_v)) / np.sqrt(np.mean(want_v ** 2)))
        # dk sums to zero: compare with the size of |dk| summed (cancellation scale)
        got_k = r["dk"][:, g].sum(axis=0)
        res[f"sum_dk_g{g}"] = float(np.max(np.abs(got_k)) / np.sqrt((r["dk"][:, g] ** 2).sum(axis=0)).max())
    return res


@pytest.mark.parametrize("config", ["C3", "C4"])
def test_fullsize_sampled_parity(config):
    from ssa_workload import CONFIGS, config_coords, make_inputs
    cfg = CONFIGS[config]
    c, grid, batch = config_coords(config)
    inp = make_inputs(c, grid, batch, cfg["H"], cfg["h_kv"], cfg["d"], "bf16", seed=cfg["seed"])
    kw = dict(h_kv=cfg["h_kv"], T=cfg["T"], m_cmp=cfg["m_cmp"], m_slc=cfg["m_slc"], m_win=cfg["m_win"],
              m_q=cfg["m_q"])
    r = run_gpu(inp, **kw)
    assert r["saved"].used_tcgen05
    plan_o = O.block_build(c, grid, batch, cfg["m_cmp"], cfg["m_slc"], cfg["m_win"], cfg["m_q"])
    assert np.array_equal(plan_o.perm, r["perm"])
    rng = np.random.Generator(np.random.PCG64(17))
    blocks = _sample_blocks(plan_o, 6 if config == "C3" else 8, rng)
    errs, n_amb = _check_blocks(inp, kw, r, plan_o, blocks)
    assert all(v <= 2e-2 for v in errs.values()), errs
    ids = _identities(inp, r, cfg["h_kv"])
    # the sums run over ~10^6 bf16-rounded gradient rows: 2e-2 of the sum's own scale
    assert all(v <= 2e-2 for v in ids.values()), ids
    print(config, "sampled blocks", blocks, errs, ids, "near-tie rows", n_amb)
