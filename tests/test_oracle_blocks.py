"""Pins for oracle O1 (block partition / sort / offsets C) — PAPER.md:143, Alg. 1 line 2.

Each pin checks the oracle against something other than itself: the SPEC worked example (golden
fixture), the m=1 special case, an independent per-token recomputation of floor(coord/m), the
contiguity and tiling invariants, and input-order invariance.
"""
import json
import os

import numpy as np
import pytest

from conftest import random_coords
from oracle import OracleError, block_build

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_spec_example_partition():
    ex = json.load(open(os.path.join(GOLD, "partition_spec_example.json")))
    c = np.array(ex["coords_bxyz"])
    m = ex["m"]
    p = block_build(c, ex["grid"], 1, m, m, m, m)
    assert p.offsets["slc"].tolist() == ex["expected_C"]
    assert p.block_coords["slc"].tolist() == ex["expected_block_coords"]
    assert p.perm.tolist() == ex["expected_sorted_original_index"]


def test_m1_singletons(rng):
    c = random_coords(rng, 50, 6)
    p = block_build(c, (6, 6, 6), 1, 1, 1, 1, 1)
    for lvl in ("cmp", "slc", "win", "q"):
        assert p.offsets[lvl].tolist() == list(range(51))


@pytest.mark.parametrize("sizes", [(4, 8, 8, 8), (2, 4, 8, 4), (4, 4, 4, 4), (2, 8, 4, 1)])
def test_per_token_recheck_and_tiling(rng, sizes):
    m_cmp, m_slc, m_win, m_q = sizes
    c = random_coords(rng, 300, 16, batch=2)
    p = block_build(c, (16, 16, 16), 2, m_cmp, m_slc, m_win, m_q)
    sc = c[p.perm]
    for lvl, m in (("cmp", m_cmp), ("slc", m_slc), ("win", m_win), ("q", m_q)):
        C = p.offsets[lvl]
        assert C[0] == 0 and C[-1] == len(c) and np.all(np.diff(C) >= 1)   # ranges tile [0,N), no empties
        for j in range(len(C) - 1):
            blk = sc[C[j]:C[j + 1]]
            # independent recomputation: every token of block j has floor(coord/m) == its block coord
            want = p.block_coords[lvl][j]
            assert np.all(blk[:, 0] == want[0])
            assert np.all(blk[:, 1:] // m == want[1:])
        # every (b, floor(coord/m)) class appears as exactly one block (contiguity)
        keys = {tuple([r[0]] + list(r[1:] // m)) for r in c}
        assert len(keys) == len(C) - 1
    # hierarchy: compression blocks nest in selection blocks
    for j, s in enumerate(p.cmp_to_slc):
        cc = p.block_coords["cmp"][j]
        ss = p.block_coords["slc"][s]
        assert cc[0] == ss[0] and np.all(cc[1:] * m_cmp // m_slc == ss[1:])
    # batch ranges
    for b in range(2):
        assert np.all(sc[p.batch_tokens[b]:p.batch_tokens[b + 1], 0] == b)


def test_selection_order_is_lexicographic(rng):
    # m_slc coarsest -> selection blocks in plain lexicographic (b, bx, by, bz) order
    c = random_coords(rng, 200, 16, batch=2)
    p = block_build(c, (16, 16, 16), 2, 4, 8, 8, 8)
    bc = [tuple(r) for r in p.block_coords["slc"]]
    assert bc == sorted(bc)


def test_order_invariance(rng):
    c = random_coords(rng, 200, 16)
    p1 = block_build(c, (16, 16, 16), 1, 4, 8, 8, 8)
    sh = rng.permutation(len(c))
    p2 = block_build(c[sh], (16, 16, 16), 1, 4, 8, 8, 8)
    assert np.array_equal(c[p1.perm], c[sh][p2.perm])
    for lvl in ("cmp", "slc"):
        assert np.array_equal(p1.offsets[lvl], p2.offsets[lvl])


def test_errors(rng):
    c = np.array([[0, 1, 1, 1], [0, 1, 1, 1]])
    with pytest.raises(OracleError):
        block_build(c, (4, 4, 4), 1, 2, 4, 4, 4)              # duplicate
    with pytest.raises(OracleError):
        block_build(np.array([[0, 4, 0, 0]]), (4, 4, 4), 1, 2, 4, 4, 4)   # out of range
    with pytest.raises(OracleError):
        block_build(np.array([[0, 1, 0, 0]]), (8, 8, 8), 1, 4, 6, 6, 6)   # 6 not multiple of 4
    with pytest.raises(OracleError):
        block_build(np.array([[0, 1, 0, 0]]), (8, 8, 8), 1, 4, 8, 6, 8)   # 6 breaks the chain


def test_nsa1d_embedding_is_fixed_length_1d_blocking():
    """The NSA-1D arm (reading R19) runs on the 3D kernels through a coordinate embedding
    (paper_2505_17412_b200.ssa.nsa1d_coords, index arithmetic only). Pinned against the oracle's direct
    1D partition: the block build of the embedded coordinates keeps the index order and its blocks are
    the fixed-length runs of l_cmp = m_cmp^3 / l_slc = m_slc^3 tokens of every batch item."""
    import oracle as O
    from paper_2505_17412_b200.ssa import nsa1d_coords
    for lengths in ([1000, 700], [512], [1, 64, 65, 1537]):
        c, grid = nsa1d_coords(lengths, 4, 8)
        plan = O.block_build(c, grid, len(lengths), 4, 8, 8, 8)
        assert np.array_equal(plan.perm, np.arange(sum(lengths)))
        assert np.array_equal(plan.offsets["cmp"], O.block_offsets_1d(lengths, 64))
        for lvl in ("slc", "win", "q"):
            assert np.array_equal(plan.offsets[lvl], O.block_offsets_1d(lengths, 512))
