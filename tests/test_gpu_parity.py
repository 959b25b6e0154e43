"""GPU parity of the whole SSA path (forward a2-a8, backward a9) through the C ABI against the float64
oracle, on the same seeded inputs (SURVEY §8c parity protocol):
  * top-k isolated: oracle top-k on the GPU's fp32 scores == GPU indices, bit for bit;
  * top-k end to end: GPU indices == oracle f64 top-k except rows inside the near-tie band;
  * outputs / gradients: oracle run with the GPU's indices; max|x-ref|/rms(ref) <= 1e-4 (fp32) or
    2e-2 (bf16 in, fp32 accumulate) — the north star's tolerances.
"""
import math

import numpy as np
import pytest

from gpu_util import rel_err, run_gpu, topk_end_to_end_check, topk_isolated_check

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2}
DELTA = {"f32": 1e-6, "bf16": 1e-4}


def _oracle(inp, I, kw, backward=True, pe=None):
    import oracle as O
    N, H, d = inp.q.shape
    f = O.ssa_forward(inp.coords, inp.grid, inp.batch, inp.q, inp.k, inp.v, inp.gates, I_override=I,
                      pe_k=None if pe is None else pe[0], pe_v=None if pe is None else pe[1], **kw)
    grads = O.ssa_backward(f, inp.q, inp.k, inp.v, inp.gates, inp.dout, h_kv=kw["h_kv"]) if backward else None
    return f, grads


def _errors(test, inp, r, f, grads, tol, backward=True, gates=None):
    """Per-tensor undiscounted errors of a GPU run `r` against oracle results (f, grads), recorded in
    the parity report. LSEs (saved log2-domain, converted to natural log) are compared in absolute
    terms against the same tolerance."""
    from gpu_util import internal_to_orig, record
    b16 = inp.dtype == "bf16"                      # out / dq / dk / dv / dgates are stored in the input dtype
    errs = {"out": record(test, "out", r["out"], f.out, tol, stored_bf16=b16)}
    for b, name in enumerate(("cmp", "slc", "win")):
        o, lse = r["saved"].branch(b)
        og = internal_to_orig(o, r["perm"])
        dc = f.o[name].shape[-1]
        if og.shape[-1] > dc:                          # d = 32 run zero-padded to 64 on tcgen05
            assert not np.any(og[..., dc:]), "padded head dims must stay zero"
            og = og[..., :dc]
        errs["o_" + name] = record(test, "o_" + name, og, f.o[name], tol)
        lg = internal_to_orig(lse, r["perm"]) * math.log(2.0)   # saved LSEs are log2-domain
        err = float(np.max(np.abs(lg - f.lse[name]))) if lg.size else 0.0
        from gpu_util import REPORT
        REPORT.append(dict(test=test, tensor="lse_" + name, n=int(lg.size), max_abs=err, rel=err, tol=tol,
                           ok=bool(err <= tol)))
        errs["lse_" + name] = err
    if backward:
        for name, g, ref in zip(("dq", "dk", "dv", "dgates"), (r["dq"], r["dk"], r["dv"], r["dgates"]), grads):
            errs[name] = record(test, name, g, ref, tol, stored_bf16=b16)
    return errs


def _check_all(inp, kw, flags=0, backward=True, pe=None, expect_tc=None, test=None):
    import os
    r = run_gpu(inp, flags=flags, backward=backward, pe=pe, **kw)
    if expect_tc is not None:
        assert r["saved"].used_tcgen05 == expect_tc
    f_free, _ = _oracle(inp, None, kw, backward=False, pe=pe)
    plan_o = f_free.plan
    assert topk_isolated_check(plan_o, r["scores"], r["I"], kw["T"]) == 0
    mism, amb = topk_end_to_end_check(plan_o, f_free.scores, r["I"], kw["T"], DELTA[inp.dtype])
    assert mism == 0, (mism, amb)
    f, grads = _oracle(inp, r["I"], kw, backward=backward, pe=pe)
    tol = TOL[inp.dtype]
    test = test or os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
    errs = _errors(test, inp, r, f, grads, tol, backward=backward)
    from gpu_util import REPORT
    REPORT.append(dict(test=test, tensor="topk", near_tie_rows=amb, mismatches=mism, ok=True))
    bad = {k: v for k, v in errs.items() if v > tol}
    assert not bad, (bad, errs)
    return r, errs


def test_c1_fp32_full():
    """BASELINE config 1: 32^3 shell (4328 tokens), 1 head d=64, blocks 4^3, T=4, fp32 fwd+bwd."""
    from ssa_workload import CONFIGS, config_coords, make_inputs
    cfg = CONFIGS["C1"]
    c, grid, batch = config_coords("C1")
    inp = make_inputs(c, grid, batch, cfg["H"], cfg["h_kv"], cfg["d"], "f32", seed=cfg["seed"])
    kw = dict(h_kv=1, T=4, m_cmp=4, m_slc=4, m_win=4, m_q=4)
    _check_all(inp, kw)


def test_c2_bf16_full():
    """BASELINE config 2: 64^3 shell (24808 tokens), 16 heads (2 kv), d=64, bf16 fwd+bwd."""
    from ssa_workload import CONFIGS, config_coords, make_inputs
    cfg = CONFIGS["C2"]
    c, grid, batch = config_coords("C2")
    inp = make_inputs(c, grid, batch, 16, 2, 64, "bf16", seed=cfg["seed"])
    kw = dict(h_kv=2, T=8, m_cmp=4, m_slc=8, m_win=8, m_q=8)
    _check_all(inp, kw, expect_tc=True)


def test_c2_fp32_full():
    """fp32 mode (the north star's 1e-4 tolerance) at BASELINE config 2's size and head layout:
    24 808 tokens, 16 heads (2 kv), d = 64 — the SIMT fp32 kernels against the oracle, undiscounted."""
    from ssa_workload import CONFIGS, config_coords, make_inputs
    c, grid, batch = config_coords("C2")
    inp = make_inputs(c, grid, batch, 16, 2, 64, "f32", seed=CONFIGS["C2"]["seed"])
    kw = dict(h_kv=2, T=8, m_cmp=4, m_slc=8, m_win=8, m_q=8)
    _check_all(inp, kw, expect_tc=False)


def test_c2_bf16_full_simt():
    """Same as test_c2_bf16_full on the SIMT kernels (SSA_FORCE_SIMT)."""
    from paper_2505_17412_b200 import ssa
    from ssa_workload import CONFIGS, config_coords, make_inputs
    c, grid, batch = config_coords("C2")
    inp = make_inputs(c, grid, batch, 16, 2, 64, "bf16", seed=CONFIGS["C2"]["seed"])
    kw = dict(h_kv=2, T=8, m_cmp=4, m_slc=8, m_win=8, m_q=8)
    _check_all(inp, kw, flags=ssa.SSA_FORCE_SIMT, expect_tc=False)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("case", ["batch3_ragged", "mq1_pertoken", "win_lt_q", "T_exceeds", "d32_hs1"])
def test_small_cases(dtype, case):
    from conftest import random_coords
    from ssa_workload import make_inputs
    rng = np.random.Generator(np.random.PCG64(hash(case) % 1000))
    H, h_kv, d = 8, 2, 64
    kw = dict(h_kv=2, T=3, m_cmp=2, m_slc=4, m_win=4, m_q=4)
    G, n, batch = 16, 500, 3
    if case == "mq1_pertoken":
        kw.update(m_q=1)
    elif case == "win_lt_q":
        kw.update(m_win=2, m_q=4)
    elif case == "T_exceeds":
        kw.update(T=64)
        G, n = 8, 120
    elif case == "d32_hs1":
        H, h_kv, d = 2, 2, 32
        kw.update(h_kv=2)
    c = random_coords(rng, n, G, batch)
    if case == "batch3_ragged":
        c = c[rng.permutation(len(c))[: len(c) - 37]]             # ragged batch items, shuffled order
    inp = make_inputs(c, (G, G, G), batch, H, h_kv, d, dtype, seed=7)
    flags = 0
    if dtype == "bf16" and case == "win_lt_q":
        # outside the tcgen05 kernels: bf16 needs the explicit SIMT opt-in (no silent fallback) ...
        from paper_2505_17412_b200 import ssa
        with pytest.raises(ssa.SSAError, match="SSA_ERR_UNSUPPORTED"):
            run_gpu(inp, backward=False, **kw)
        flags = ssa.SSA_FORCE_SIMT
    _check_all(inp, kw, flags=flags)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_single_token(dtype):
    from ssa_workload import make_inputs
    c = np.array([[0, 3, 4, 5]], dtype=np.int32)
    inp = make_inputs(c, (8, 8, 8), 1, 4, 2, 64, dtype, seed=3)
    kw = dict(h_kv=2, T=8, m_cmp=4, m_slc=8, m_win=8, m_q=8)
    _check_all(inp, kw)


def test_pe_tables():
    from conftest import random_coords
    from ssa_workload import make_inputs, round_to_bf16
    rng = np.random.Generator(np.random.PCG64(9))
    c = random_coords(rng, 400, 16, 1)
    inp = make_inputs(c, (16, 16, 16), 1, 4, 2, 64, "f32", seed=1)
    pe = (rng.standard_normal((64, 2, 64)).astype(np.float32), rng.standard_normal((64, 2, 64)).astype(np.float32))
    _check_all(inp, dict(h_kv=2, T=3, m_cmp=4, m_slc=8, m_win=8, m_q=8), pe=pe)


def test_planted_selection_bit_exact():
    """Planted workload: the top-T gap is large, so GPU indices must equal the oracle's exactly."""
    import oracle as O
    from ssa_workload import config_coords, make_inputs, planted_inputs
    c, grid, batch = config_coords("C1", shapes=[(32, 13.0, 2.0)])
    inp = make_inputs(c, grid, batch, 8, 2, 64, "bf16", seed=4)
    inp = planted_inputs(inp, m_q=8, m_slc=8, T=4, h_s=4)
    kw = dict(h_kv=2, T=4, m_cmp=4, m_slc=8, m_win=8, m_q=8)
    r = run_gpu(inp, backward=False, **kw)
    f = O.ssa_forward(inp.coords, inp.grid, inp.batch, inp.q, inp.k, inp.v, inp.gates, **kw)
    assert np.array_equal(r["I"], f.I)


def test_gpu_sorted_input_flag():
    """SSA_INPUT_SORTED: feeding block-sorted tensors gives the same (sorted) result."""
    import torch
    from conftest import random_coords
    from gpu_util import to_dev
    from paper_2505_17412_b200 import ssa
    from ssa_workload import make_inputs
    rng = np.random.Generator(np.random.PCG64(2))
    c = random_coords(rng, 300, 16, 2)
    inp = make_inputs(c, (16, 16, 16), 2, 4, 2, 64, "bf16", seed=2)
    kw = dict(h_kv=2, T=3, m_cmp=2, m_slc=4, m_win=4, m_q=4)
    r = run_gpu(inp, backward=False, **kw)
    perm = r["perm"]
    plan = r["plan"]
    cfg = ssa.AttnCfg(h_q=4, h_kv=2, d=64, top_k=3, dtype=torch.bfloat16, flags=ssa.SSA_INPUT_SORTED)
    q, k, v, g = (to_dev(x[perm], torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates))
    out, _ = ssa.ssa_forward(plan, cfg, q, k, v, g)
    assert np.array_equal(out.float().cpu().numpy(), r["out"][perm].astype(np.float32))


@pytest.mark.parametrize("heads", [(8, 1), (32, 4), (4, 4), (16, 16)])
def test_tc_head_layouts(heads):
    """tcgen05 path with other GQA layouts (h_s = H / h_kv = 8, 8, 1, 1): the rows of a query block are
    tokens x h_s, so 128-row tiles hold 16 or 128 tokens; parity and top-k as for C2."""
    from ssa_workload import batch_coords, make_inputs, sphere_shell
    H, h_kv = heads
    c = batch_coords([sphere_shell(32, 13.0, 2.0)])
    inp = make_inputs(c, (32, 32, 32), 1, H, h_kv, 64, "bf16", seed=5)
    kw = dict(h_kv=h_kv, T=4, m_cmp=4, m_slc=8, m_win=8, m_q=8)
    _check_all(inp, kw, expect_tc=True)


@pytest.mark.parametrize("m_q", [1, 2])
@pytest.mark.parametrize("heads", [(8, 2), (4, 4), (32, 2)])
def test_tc_small_query_heads(heads, m_q):
    """Per-token / small query blocks with other head layouts (h_s = 4, 1, 16 rows per token): tokens that
    are not a multiple of the 8-row granule leave padded slots in the KV-outer packed row tiles (valid
    counts < 8, TMA boxes reading the next token's rows, masked by an LSE of +inf), and h_s = 1 puts 128
    tokens in a row tile of the virtual query level — parity and top-k against the oracle."""
    from ssa_workload import batch_coords, make_inputs, sphere_shell
    H, h_kv = heads
    c = batch_coords([sphere_shell(32, 13.0, 2.0)])
    inp = make_inputs(c, (32, 32, 32), 1, H, h_kv, 64, "bf16", seed=31)
    kw = dict(h_kv=h_kv, T=4, m_cmp=4, m_slc=8, m_win=8, m_q=m_q)
    _check_all(inp, kw, expect_tc=True, test=f"test_tc_small_query_heads[{H},{h_kv},{m_q}]")


@pytest.mark.parametrize("T", [4, 32])
def test_tc_dense_blocks(T):
    """Solid ball (5 616 tokens): a full 8^3 selection block of 512 keys (4 tiles) among blocks of 47-416
    keys, so packed key tiles hold segments of 64-row boxes that cross tile boundaries; T = 32 exceeds the
    27 selection blocks (-1 padding) — tcgen05 path against the oracle."""
    from ssa_workload import batch_coords, make_inputs
    G, r = 24, 11.0
    ax = np.arange(G)
    X, Y, Z = np.meshgrid(ax, ax, ax, indexing="ij")
    ball = np.stack([X, Y, Z], -1)[(X - 11.5) ** 2 + (Y - 11.5) ** 2 + (Z - 11.5) ** 2 <= r * r].astype(np.int32)
    c = batch_coords([ball])
    inp = make_inputs(c, (G, G, G), 1, 8, 2, 64, "bf16", seed=13)
    kw = dict(h_kv=2, T=T, m_cmp=4, m_slc=8, m_win=8, m_q=8)
    r_, _ = _check_all(inp, kw, expect_tc=True)
    assert (r_["I"] < 0).any() == (T > 27)


def _shell_case(H=16, h_kv=2, seed=21):
    from ssa_workload import batch_coords, make_inputs, sphere_shell
    c = batch_coords([sphere_shell(32, 13.0, 2.0)])
    inp = make_inputs(c, (32, 32, 32), 1, H, h_kv, 64, "bf16", seed=seed)
    return inp, dict(h_kv=h_kv, T=4, m_cmp=4, m_slc=8, m_win=8, m_q=8)


@pytest.mark.parametrize("dscale", [1e-6, 1e-9, 3e3])
def test_dout_scale(dscale):
    """the tcgen05 backward's MMA operands for dO are fp16. A loss averaged over ~1e5
    tokens gives dO ~ 1e-6 and below, where an unscaled fp16 copy loses bits (< 6e-5) or flushes to zero
    (< 6e-8). The row prologue scales dO by a power of two from max|dO| (exact), the epilogues undo it:
    relative accuracy must not depend on the magnitude of dO."""
    from ssa_workload import round_to_bf16
    inp, kw = _shell_case()
    inp.dout = round_to_bf16(inp.dout * dscale)
    _check_all(inp, kw, expect_tc=True, test=f"test_dout_scale[{dscale}]")


def test_negative_controls():
    """The parity checks have teeth: with the GPU result unchanged, (1) one selected index
    swapped for an unselected block, (2) the cmp / slc gates swapped, (3) a perturbed saved LSE fed to
    the GPU backward, and (4) one perturbed GPU score in the isolated top-k check must each FAIL the same
    comparisons that pass on the true state."""
    import torch
    from gpu_util import to_dev
    from paper_2505_17412_b200 import ssa
    inp, kw = _shell_case(H=8, seed=22)
    tol = TOL["bf16"]
    r = run_gpu(inp, **kw)
    f, grads = _oracle(inp, r["I"], kw)
    base = _errors("negctl:base", inp, r, f, grads, tol)
    assert max(base.values()) <= tol, base
    plan_o = f.plan
    # (1) perturbed index
    I_bad = r["I"].copy()
    Q, g = 5, 1
    b = int(plan_o.sorted_coords[int(plan_o.offsets["q"][Q]), 0])
    s0, s1 = int(plan_o.batch_blocks["slc"][b]), int(plan_o.batch_blocks["slc"][b + 1])
    unsel = [B for B in range(s0, s1) if B not in set(I_bad[Q, g].tolist())]
    I_bad[Q, g, 0] = unsel[len(unsel) // 2]
    I_bad[Q, g] = np.sort(I_bad[Q, g])
    f1, g1 = _oracle(inp, I_bad, kw)
    e1 = _errors("negctl:index", inp, r, f1, g1, tol)
    assert e1["o_slc"] > tol and e1["out"] > tol, e1
    # (2) swapped gates (cmp <-> slc)
    from dataclasses import replace
    inp2 = replace(inp, gates=inp.gates[..., [1, 0, 2]].copy())
    f2, g2 = _oracle(inp2, r["I"], kw)
    e2 = _errors("negctl:gates", inp, r, f2, g2, tol)
    assert e2["out"] > tol and e2["dq"] > tol, e2        # (dgates = <dO, O_c> does not involve the gates)
    # (3) perturbed saved LSE (selection branch, one query block's rows, +0.25 in log2 units) -> GPU backward
    o_slc, lse_slc = r["saved"].branch(1)
    a, e = int(plan_o.offsets["q"][Q]), int(plan_o.offsets["q"][Q + 1])
    lse_slc[:, a:e] += 0.25
    q, k, v, gt, do = (to_dev(x, torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout))
    dq3, dk3, dv3, _ = ssa.ssa_backward(r["plan"], r["cfg"], r["saved"], q, k, v, gt, do)
    torch.cuda.synchronize()
    r3 = dict(r, dq=dq3.float().cpu().numpy().astype(np.float64), dk=dk3.float().cpu().numpy().astype(np.float64),
              dv=dv3.float().cpu().numpy().astype(np.float64))
    e3 = _errors("negctl:lse", inp, r3, f, grads, tol)
    assert e3["lse_slc"] > tol and e3["dq"] > tol, e3
    # (4) one perturbed score in the isolated top-k check
    sc = r["scores"].copy()
    j = int(unsel[0]) - s0
    sc[Q, g, j] = sc[Q, g, :s1 - s0].max() * 2
    assert topk_isolated_check(plan_o, sc, r["I"], kw["T"]) >= 1


def test_nsa1d_arm():
    """The NSA-1D blocking arm (reading R19): fixed-length 1D blocks of 64 / 512 consecutive
    tokens through ssa.nsa1d_coords on the unchanged tcgen05 kernels — plan = the oracle's 1D partition,
    parity of the whole step against the oracle on the same (embedded) coordinates."""
    import oracle as O
    from paper_2505_17412_b200 import ssa
    from ssa_workload import make_inputs
    lengths = [3000, 1700]
    c, grid = ssa.nsa1d_coords(lengths, 4, 8)
    inp = make_inputs(c, grid, 2, 16, 2, 64, "bf16", seed=23)
    kw = dict(h_kv=2, T=4, m_cmp=4, m_slc=8, m_win=8, m_q=8)
    r, _ = _check_all(inp, kw, expect_tc=True, test="test_nsa1d_arm")
    assert np.array_equal(r["perm"], np.arange(sum(lengths)))
    assert np.array_equal(r["plan"].offsets(ssa.LEVEL_CMP).cpu().numpy(), O.block_offsets_1d(lengths, 64))
    assert np.array_equal(r["plan"].offsets(ssa.LEVEL_SLC).cpu().numpy(), O.block_offsets_1d(lengths, 512))


def test_paper_head_layout_d32():
    """The paper's DiT attention layout: 2 kv groups x 16 heads, head dim 32 — on the tcgen05
    kernels (heads zero-padded to 64 inside the library), parity against the oracle at d = 32."""
    from ssa_workload import batch_coords, make_inputs, sphere_shell
    c = batch_coords([sphere_shell(32, 13.0, 2.0)])
    inp = make_inputs(c, (32, 32, 32), 1, 32, 2, 32, "bf16", seed=24)
    kw = dict(h_kv=2, T=4, m_cmp=4, m_slc=8, m_win=8, m_q=8)
    r, _ = _check_all(inp, kw, expect_tc=True, test="test_paper_head_layout_d32")
    assert r["saved"].d_internal == 64


# query-level choices of the tcgen05 path for m_q < m_slc (pertoken.cu knobs): the plan's own choice,
# the query-block tiles as they are, the virtual level for dQ / selection only, and for the KV-outer too
_VQ_MODES = {
    "auto": {},
    "direct": {"SSA_VQ": "0"},
    "vq_dq": {"SSA_VQ_ROWS": "100000", "SSA_VQ_KV_ROWS": "0.001"},
    "vq_all": {"SSA_VQ_ROWS": "100000", "SSA_VQ_KV_ROWS": "100000", "SSA_VQ_QB_PER_ITEM": "3"},
    "union": {"SSA_VQ_BLOCKSEL": "0"},       # m_q = 1 through the union-masked sub-groups
    "blocks": {"SSA_VQ_BLOCKSEL": "2"},      # the per-block selection passes also for m_q = 2, 4
}


@pytest.mark.parametrize("mode", list(_VQ_MODES))
@pytest.mark.parametrize("m_q", [1, 2, 4])
def test_tc_small_query_blocks(m_q, mode, monkeypatch):
    """Query blocks smaller than the selection blocks on the tcgen05 kernels — m_q = 1 is the paper's
    per-token selection, I in R^{N x h_kv x T} (Alg. 1): every token's
    Eq. 8 score is its own (8 heads), its top-T its own; the window is the m_win^3 block holding the
    query block. Parity (top-k isolated / end to end, every output and gradient) against the oracle, for
    each query-level choice of the kernels (same arithmetic per row, only the row / key grouping differs;
    vq_all also splits every key's rows into many KV-outer work items)."""
    from ssa_workload import batch_coords, make_inputs, sphere_shell
    for k, v in _VQ_MODES[mode].items():
        monkeypatch.setenv(k, v)
    c = batch_coords([sphere_shell(32, 13.0, 2.0)])
    inp = make_inputs(c, (32, 32, 32), 1, 16, 2, 64, "bf16", seed=25)
    kw = dict(h_kv=2, T=4, m_cmp=4, m_slc=8, m_win=8, m_q=m_q)
    _check_all(inp, kw, expect_tc=True, test=f"test_tc_small_query_blocks[{m_q},{mode}]")
