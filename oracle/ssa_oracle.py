"""Float64 CPU oracle of Spatial Sparse Attention (Direct3D-S2, arXiv 2505.17412, §4.1).

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import or execute anything under `oracle/`. The product path
(`paper_2505_17412_b200/`) never imports it, and this module imports nothing from the product path:
the two share no code (task rule ③). Inputs come from `ssa_workload` (random numbers only).

Plain, slow, obviously-correct numpy float64. Each function cites the passage of
/root/reference/PAPER.md ("P:<line>") it follows; readings where the paper is silent or garbled are
marked READING and listed in DESIGN.md §"Readings". Library primitives used as single steps: numpy
sort (python `sorted`), matmul, exp/log, max.

Conventions
  * coords: int [N,4] rows (b, x, y, z); grid (Gx, Gy, Gz); batch items never interact.
  * heads: q [N, H, d] with H = h_kv * h_s, head h = g*h_s + s attends kv head g (GQA, Alg. 1
    signature P:182); k, v [N, h_kv, d]; gates [N, H, 3] in Eq. 6 order (cmp, slc, win).
  * scale = 1/sqrt(d) (Eq. 5). LSE is the natural log of sum exp(scale * q.k).
  * all outputs are returned in the ORIGINAL token order unless the name says "sorted".

Parity status: every function here is pinned by `tests/test_oracle_*.py` (closed forms, brute force,
special cases reducing to full attention, finite differences, SPEC worked examples); none is
"parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

LEVELS = ("cmp", "slc", "win", "q")


class OracleError(ValueError):
    """Invalid input (duplicate coordinate, out-of-range coordinate, invalid block hierarchy...)."""


# --------------------------------------------------------------------------------------------------
# O1. Spatial block partition + sort + offsets C.  P:143 ("divide the 3D space into subgrids of size
# m^3, where active tokens ... residing in the same subgrid are grouped into one block"), P:175 ("first
# sort the input tokens based on their block indices, then compute the starting index C of each block"),
# Alg. 1 line 2. P:166: "m_slc must be both greater than and divisible by m_cmp".
# READING R1: sort key is hierarchical-lexicographic over the distinct block sizes, coarse to fine,
# then voxel-in-finest-block; every level is then contiguous in the sorted order. R2: the chain is
# relaxed to >= (so config C1, all sizes 4, is legal). R3: empty blocks are never materialised.
# --------------------------------------------------------------------------------------------------
@dataclass
class BlockPlan:
    N: int
    batch: int
    grid: tuple
    sizes: dict                 # level -> m
    perm: np.ndarray            # [N] sorted position -> original index
    inv_perm: np.ndarray        # [N] original index -> sorted position
    sorted_coords: np.ndarray   # [N,4]
    offsets: dict               # level -> C [N_l+1] (token offsets in sorted order)
    block_coords: dict          # level -> [N_l,4] (b, bx, by, bz)
    tok_block: dict             # level -> [N] block id of each SORTED token
    batch_blocks: dict          # level -> [batch+1] first block of each batch item
    batch_tokens: np.ndarray    # [batch+1] first sorted token of each batch item
    cmp_to_slc: np.ndarray      # [N_cmp] enclosing selection block of each compression block

    def n_blocks(self, level: str) -> int:
        return int(self.offsets[level].shape[0] - 1)


def _chain(sizes: dict) -> list:
    ms = sorted(set(int(m) for m in sizes.values()), reverse=True)
    for a, b in zip(ms, ms[1:]):
        if a % b != 0:
            raise OracleError(f"block sizes {ms} do not form a divisibility chain")
    return ms


def block_build(coords, grid, batch: int, m_cmp: int, m_slc: int, m_win: int, m_q: int) -> BlockPlan:
    coords = np.asarray(coords, dtype=np.int64).reshape(-1, 4)
    N = coords.shape[0]
    sizes = dict(cmp=int(m_cmp), slc=int(m_slc), win=int(m_win), q=int(m_q))
    if min(sizes.values()) < 1:
        raise OracleError("block sizes must be >= 1")
    if m_slc < m_cmp or m_slc % m_cmp != 0:          # P:166 (relaxed to >=, READING R2)
        raise OracleError("m_slc must be a multiple of m_cmp")
    ms = _chain(sizes)
    G = tuple(int(g) for g in grid)
    if N:
        if coords[:, 0].min() < 0 or coords[:, 0].max() >= batch:
            raise OracleError("batch index out of range")
        for a in range(3):
            if coords[:, 1 + a].min() < 0 or coords[:, 1 + a].max() >= G[a]:
                raise OracleError("coordinate out of range")
    if len(set(map(tuple, coords.tolist()))) != N:
        raise OracleError("duplicate coordinates")

    def key(c):
        b, x, y, z = (int(t) for t in c)
        m0 = ms[0]
        kk = [b, x // m0, y // m0, z // m0]
        for hi, lo in zip(ms, ms[1:]):
            r = hi // lo
            kk += [(x // lo) % r, (y // lo) % r, (z // lo) % r]
        ml = ms[-1]
        kk += [x % ml, y % ml, z % ml]
        return tuple(kk)

    perm = np.array(sorted(range(N), key=lambda i: key(coords[i])), dtype=np.int64)
    inv_perm = np.empty(N, dtype=np.int64)
    inv_perm[perm] = np.arange(N)
    sc = coords[perm]
    offsets, bcoords, tokb, bblocks = {}, {}, {}, {}
    for lvl, m in sizes.items():
        blk = np.concatenate([sc[:, :1], sc[:, 1:] // m], axis=1)
        starts = [i for i in range(N) if i == 0 or tuple(blk[i]) != tuple(blk[i - 1])]
        C = np.array(starts + [N], dtype=np.int64)
        ids = np.zeros(N, dtype=np.int64)
        for j in range(len(starts)):
            ids[C[j]:C[j + 1]] = j
        offsets[lvl] = C
        bcoords[lvl] = blk[np.array(starts, dtype=np.int64)] if starts else np.zeros((0, 4), np.int64)
        tokb[lvl] = ids
        bb = np.zeros(batch + 1, dtype=np.int64)
        for b in range(batch + 1):
            bb[b] = int(np.searchsorted(bcoords[lvl][:, 0], b, side="left")) if starts else 0
        bblocks[lvl] = bb
    bt = np.array([int(np.searchsorted(sc[:, 0], b, side="left")) for b in range(batch + 1)], np.int64)
    n_cmp = len(offsets["cmp"]) - 1
    cmp_to_slc = np.array([tokb["slc"][offsets["cmp"][j]] for j in range(n_cmp)], dtype=np.int64)
    return BlockPlan(N=N, batch=batch, grid=G, sizes=sizes, perm=perm, inv_perm=inv_perm,
                     sorted_coords=sc, offsets=offsets, block_coords=bcoords, tok_block=tokb,
                     batch_blocks=bblocks, batch_tokens=bt, cmp_to_slc=cmp_to_slc)


# --------------------------------------------------------------------------------------------------
# Dense attention, Eqs. 4-5: o_t = sum_i p_ti v_i / sum_j p_tj, p_tj = exp(q_t.k_j/sqrt(d)).
# Evaluated with the row max subtracted (same value). Returns o and the natural-log LSE.
# --------------------------------------------------------------------------------------------------
def dense_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float):
    """q [R,d], k [M,d], v [M,dv] -> (o [R,dv], lse [R], p [R,M])."""
    s = scale * (np.asarray(q, np.float64) @ np.asarray(k, np.float64).T)
    mx = s.max(axis=1, keepdims=True)
    e = np.exp(s - mx)
    den = e.sum(axis=1, keepdims=True)
    p = e / den
    o = p @ np.asarray(v, np.float64)
    lse = (mx + np.log(den))[:, 0]
    return o, lse, p


def dense_attention_backward(q, k, v, p, o, do, scale):
    """Analytic gradient of dense_attention: returns (dq, dk, dv) for one (rows x keys) problem."""
    q, k, v, p, o, do = (np.asarray(t, np.float64) for t in (q, k, v, p, o, do))
    dv = p.T @ do
    dp = do @ v.T
    dsum = (do * o).sum(axis=1, keepdims=True)
    ds = p * (dp - dsum)
    dq = scale * ds @ k
    dk = scale * ds.T @ q
    return dq, dk, dv


# --------------------------------------------------------------------------------------------------
# O2. Sparse 3D compression, Eq. 7: k^cmp = delta(k + PE(k)), delta = "sparse 3D
# convolution followed by sparse 3D mean pooling". READING R4: the learned convolution weights are
# unavailable -> delta = masked mean pool over the active tokens of each m_cmp^3 block; PE is an
# optional caller table indexed by the intra-block offset (x%m, y%m, z%m) ("intra-block positional
# encoding"). READING R5: v^cmp is formed the same way as k^cmp.
# --------------------------------------------------------------------------------------------------
def local_index(sorted_coords: np.ndarray, m: int) -> np.ndarray:
    c = sorted_coords[:, 1:] % m
    return (c[:, 0] * m + c[:, 1]) * m + c[:, 2]


def compress(plan: BlockPlan, x_sorted: np.ndarray, pe: np.ndarray | None = None) -> np.ndarray:
    """x_sorted [N, h_kv, d] -> [N_cmp, h_kv, d] block means (plus optional PE table [m^3, h_kv, d])."""
    x = np.asarray(x_sorted, np.float64)
    if pe is not None:
        x = x + np.asarray(pe, np.float64)[local_index(plan.sorted_coords, plan.sizes["cmp"])]
    C = plan.offsets["cmp"]
    out = np.zeros((len(C) - 1,) + x.shape[1:], np.float64)
    for j in range(len(C) - 1):
        out[j] = x[C[j]:C[j + 1]].mean(axis=0)
    return out


# --------------------------------------------------------------------------------------------------
# Branch attentions (Eq. 6) for one (query block, kv group) at a time.
# Rows of a query block Q and group g are the pairs (t, s), t in Q, s < h_s, ordered t-major.
# --------------------------------------------------------------------------------------------------
def _rows(q_sorted, t0, t1, g, h_s):
    return np.asarray(q_sorted[t0:t1, g * h_s:(g + 1) * h_s, :], np.float64).reshape(-1, q_sorted.shape[2])


def compression_attention(plan: BlockPlan, q_sorted, k_cmp, v_cmp, h_kv: int, scale: float):
    """Eq. 6 term 1: each query attends every compression block of its batch item.
    READING R6: non-causal, all blocks of the batch item, own block included.
    Returns sorted-order o [N,H,d], lse [N,H] and, per (query block, g), the probability matrix
    P [rows, N_cmp(b)] needed by Eq. 8."""
    N, H, d = q_sorted.shape
    h_s = H // h_kv
    o = np.zeros((N, H, v_cmp.shape[2]))
    lse = np.zeros((N, H))
    probs = {}
    Cq = plan.offsets["q"]
    for Q in range(len(Cq) - 1):
        t0, t1 = int(Cq[Q]), int(Cq[Q + 1])
        b = int(plan.sorted_coords[t0, 0])
        c0, c1 = int(plan.batch_blocks["cmp"][b]), int(plan.batch_blocks["cmp"][b + 1])
        for g in range(h_kv):
            oo, ll, pp = dense_attention(_rows(q_sorted, t0, t1, g, h_s), k_cmp[c0:c1, g], v_cmp[c0:c1, g], scale)
            o[t0:t1, g * h_s:(g + 1) * h_s] = oo.reshape(t1 - t0, h_s, -1)
            lse[t0:t1, g * h_s:(g + 1) * h_s] = ll.reshape(t1 - t0, h_s)
            probs[(Q, g)] = pp
    return o, lse, probs


# --------------------------------------------------------------------------------------------------
# O4. Selection-block scores, Eq. 8: s^slc_t = sum_{i in B_cmp} sum_{h=1}^{h_s} s^{cmp,i}_{t,h}.
# READING R7: s^cmp are post-softmax probabilities of the compression attention. READING R8 (query-
# block granularity): the score of query block Q is the sum of Eq. 8 over the tokens t in Q; m_q = 1
# (one token per block, coords unique) is exactly the paper's per-token Eq. 8.
# --------------------------------------------------------------------------------------------------
def block_scores(plan: BlockPlan, probs: dict, h_kv: int) -> dict:
    """-> {(Q, g): scores [N_slc(b)] over the selection blocks of Q's batch item (local index)}."""
    Cq = plan.offsets["q"]
    out = {}
    for Q in range(len(Cq) - 1):
        b = int(plan.sorted_coords[int(Cq[Q]), 0])
        c0, c1 = int(plan.batch_blocks["cmp"][b]), int(plan.batch_blocks["cmp"][b + 1])
        s0, s1 = int(plan.batch_blocks["slc"][b]), int(plan.batch_blocks["slc"][b + 1])
        for g in range(h_kv):
            p = probs[(Q, g)]                       # [rows = |Q| * h_s, N_cmp(b)]
            per_cmp = p.sum(axis=0)                 # sum over t in Q and the h_s shared heads
            sc = np.zeros(s1 - s0)
            for i in range(c0, c1):                 # sum over compression blocks inside each slc block
                sc[int(plan.cmp_to_slc[i]) - s0] += per_cmp[i - c0]
            out[(Q, g)] = sc
    return out


# --------------------------------------------------------------------------------------------------
# O5. Top-k ("the top-k selection blocks with the highest scores are selected").
# READING R9: T is a parameter (paper silent); effective T = min(T, N_slc(b)); ties -> lower block
# index; no forced own block; output ascending by block index, padded with -1.
# --------------------------------------------------------------------------------------------------
def topk_select(scores: np.ndarray, T: int, base: int = 0) -> np.ndarray:
    n = scores.shape[0]
    order = sorted(range(n), key=lambda i: (-float(scores[i]), i))
    chosen = sorted(order[:min(T, n)])
    out = np.full(T, -1, dtype=np.int64)
    out[:len(chosen)] = np.array(chosen, dtype=np.int64) + base
    return out


def topk_all(plan: BlockPlan, scores: dict, h_kv: int, T: int) -> np.ndarray:
    Cq = plan.offsets["q"]
    I = np.full((len(Cq) - 1, h_kv, T), -1, dtype=np.int64)
    for (Q, g), sc in scores.items():
        b = int(plan.sorted_coords[int(Cq[Q]), 0])
        I[Q, g] = topk_select(sc, T, base=int(plan.batch_blocks["slc"][b]))
    return I


# --------------------------------------------------------------------------------------------------
# O6. Spatial blockwise selection attention — Algorithm 1, literally, per token t.
# READINGS (Alg. 1 garbles): R10 l is initialised to -inf, not 0 (P:191 vs the LSE update P:207);
# R11 the 1/sqrt(d) scale of Eq. 5 is applied to s (P:199 omits it); R12 the last B_k chunk is
# clipped at b_e; selection uses I of the query block containing t (R8).
# --------------------------------------------------------------------------------------------------
def selection_attention_alg1(plan: BlockPlan, q_sorted, k_sorted, v_sorted, I, h_kv: int, scale: float,
                             B_k: int = 64):
    N, H, d = q_sorted.shape
    h_s = H // h_kv
    C = plan.offsets["slc"]
    o_all = np.zeros((N, H, v_sorted.shape[2]))
    l_all = np.zeros((N, H))
    for t in range(N):                                           # line 3
        Q = int(plan.tok_block["q"][t])
        for h in range(h_kv):                                    # line 4
            o = np.zeros((h_s, v_sorted.shape[2]))               # line 5
            l = np.full(h_s, -np.inf)                            # line 5 (READING R10)
            m = np.full(h_s, -np.inf)
            qt = np.asarray(q_sorted[t, h * h_s:(h + 1) * h_s], np.float64)   # line 6
            for j in range(I.shape[2]):                          # line 7
                blk = int(I[Q, h, j])
                if blk < 0:
                    continue
                b_s, b_e = int(C[blk]), int(C[blk + 1]) - 1      # line 8
                for i in range(b_s, b_e + 1, B_k):               # line 9
                    i1 = min(i + B_k, b_e + 1)                   # READING R12
                    ki = np.asarray(k_sorted[i:i1, h], np.float64)     # line 10
                    vi = np.asarray(v_sorted[i:i1, h], np.float64)
                    s = scale * qt @ ki.T                        # line 11 (READING R11)
                    m_new = np.maximum(m, s.max(axis=1))         # line 12
                    p = np.exp(s - m_new[:, None])               # line 13
                    o = np.exp(m - m_new)[:, None] * o + p @ vi  # line 14
                    l = m_new + np.log(np.exp(l - m_new) + p.sum(axis=1))   # line 15
                    m = m_new
            o = np.exp(m - l)[:, None] * o                       # line 18
            o_all[t, h * h_s:(h + 1) * h_s] = o                  # line 19
            l_all[t, h * h_s:(h + 1) * h_s] = l
    return o_all, l_all


def _selected_tokens(plan: BlockPlan, I, Q, g):
    C = plan.offsets["slc"]
    idx = [np.arange(C[b], C[b + 1]) for b in I[Q, g] if b >= 0]
    return np.concatenate(idx) if idx else np.zeros(0, dtype=np.int64)


def selection_attention(plan: BlockPlan, q_sorted, k_sorted, v_sorted, I, h_kv: int, scale: float):
    """Same function as Alg. 1 written as dense attention (Eqs. 4-5) over the concatenated tokens of
    the selected blocks ("all tokens contained within them are concatenated")."""
    N, H, d = q_sorted.shape
    h_s = H // h_kv
    o = np.zeros((N, H, v_sorted.shape[2]))
    lse = np.zeros((N, H))
    Cq = plan.offsets["q"]
    for Q in range(len(Cq) - 1):
        t0, t1 = int(Cq[Q]), int(Cq[Q + 1])
        for g in range(h_kv):
            kt = _selected_tokens(plan, I, Q, g)
            oo, ll, _ = dense_attention(_rows(q_sorted, t0, t1, g, h_s), k_sorted[kt, g], v_sorted[kt, g], scale)
            o[t0:t1, g * h_s:(g + 1) * h_s] = oo.reshape(t1 - t0, h_s, -1)
            lse[t0:t1, g * h_s:(g + 1) * h_s] = ll.reshape(t1 - t0, h_s)
    return o, lse


# --------------------------------------------------------------------------------------------------
# O7. Sparse 3D window: "partition the input token-containing voxels into non-overlapping
# windows of size m_win^3 ... localized self-attention ... exclusively over this constructed token
# subset". READING R13: windows aligned at the origin, unshifted.
# --------------------------------------------------------------------------------------------------
def window_attention(plan: BlockPlan, q_sorted, k_sorted, v_sorted, h_kv: int, scale: float):
    N, H, d = q_sorted.shape
    h_s = H // h_kv
    o = np.zeros((N, H, v_sorted.shape[2]))
    lse = np.zeros((N, H))
    Cw = plan.offsets["win"]
    for w in range(len(Cw) - 1):
        t0, t1 = int(Cw[w]), int(Cw[w + 1])
        for g in range(h_kv):
            oo, ll, _ = dense_attention(_rows(q_sorted, t0, t1, g, h_s), k_sorted[t0:t1, g], v_sorted[t0:t1, g], scale)
            o[t0:t1, g * h_s:(g + 1) * h_s] = oo.reshape(t1 - t0, h_s, -1)
            lse[t0:t1, g * h_s:(g + 1) * h_s] = ll.reshape(t1 - t0, h_s)
    return o, lse


# --------------------------------------------------------------------------------------------------
# O8. Gated combination, Eq. 6. READING R14: gates are given per (token, head, branch)
# (already post-sigmoid); a per-token gate is the special case of equal values over heads.
# --------------------------------------------------------------------------------------------------
def gate_combine(o_cmp, o_slc, o_win, gates):
    g = np.asarray(gates, np.float64)
    return g[..., 0:1] * o_cmp + g[..., 1:2] * o_slc + g[..., 2:3] * o_win


# --------------------------------------------------------------------------------------------------
# Full forward (Fig. "SSA" caption P:121, Eq. 6) and backward.
# --------------------------------------------------------------------------------------------------
@dataclass
class ForwardResult:
    out: np.ndarray       # [N,H,d] original order
    o: dict               # branch -> [N,H,d] original order
    lse: dict             # branch -> [N,H]  original order
    I: np.ndarray         # [N_q, h_kv, T] global slc block ids
    scores: dict          # (Q,g) -> [N_slc(b)]
    k_cmp: np.ndarray     # [N_cmp, h_kv, d]
    v_cmp: np.ndarray
    plan: BlockPlan


def ssa_forward(coords, grid, batch, q, k, v, gates, *, h_kv, T, m_cmp, m_slc, m_win, m_q,
                scale=None, pe_k=None, pe_v=None, I_override=None, plan=None) -> ForwardResult:
    """SSA forward. `I_override` lets a parity test feed the GPU's selected indices
    so that near-tie index flips cannot pollute the numeric comparison."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    N, H, d = q.shape
    if H % h_kv:
        raise OracleError("H must be a multiple of h_kv")
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    if plan is None:
        plan = block_build(coords, grid, batch, m_cmp, m_slc, m_win, m_q)
    P = plan.perm
    qs, ks, vs, gs = q[P], k[P], v[P], np.asarray(gates, np.float64)[P]
    k_cmp = compress(plan, ks, pe_k)
    v_cmp = compress(plan, vs, pe_v)
    o_c, l_c, probs = compression_attention(plan, qs, k_cmp, v_cmp, h_kv, scale)
    scores = block_scores(plan, probs, h_kv)
    I = topk_all(plan, scores, h_kv, T) if I_override is None else np.asarray(I_override, np.int64)
    o_s, l_s = selection_attention(plan, qs, ks, vs, I, h_kv, scale)
    o_w, l_w = window_attention(plan, qs, ks, vs, h_kv, scale)
    out = gate_combine(o_c, o_s, o_w, gs)
    inv = plan.inv_perm
    return ForwardResult(out=out[inv], o=dict(cmp=o_c[inv], slc=o_s[inv], win=o_w[inv]),
                         lse=dict(cmp=l_c[inv], slc=l_s[inv], win=l_w[inv]), I=I, scores=scores,
                         k_cmp=k_cmp, v_cmp=v_cmp, plan=plan)


def ssa_backward(fwd: ForwardResult, q, k, v, gates, dout, *, h_kv, scale=None):
    """Analytic gradients of ssa_forward with the block structure and the selected indices I held
    constant (hard routing; READING R15 — the paper gives no backward, P:391 reports only its speed).
    dgate_c = <dO, O_c>; per branch dO_c = omega_c dO; softmax backward dS = P (dP - <dO_c, O_c>);
    the compression branch chains through the mean pool: dk_j += dk^cmp_{B(j)} / n_B (PE constant).
    Returns (dq, dk, dv, dgates) in original order."""
    plan = fwd.plan
    q = np.asarray(q, np.float64)
    N, H, d = q.shape
    h_s = H // h_kv
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    P = plan.perm
    qs = q[P]
    ks = np.asarray(k, np.float64)[P]
    vs = np.asarray(v, np.float64)[P]
    gs = np.asarray(gates, np.float64)[P]
    dos = np.asarray(dout, np.float64)[P]
    o = {c: fwd.o[c][P] for c in fwd.o}
    dgates = np.stack([(dos * o[c]).sum(axis=2) for c in ("cmp", "slc", "win")], axis=2)
    dq = np.zeros_like(qs)
    dk = np.zeros_like(ks)
    dv = np.zeros_like(vs)
    dk_cmp = np.zeros_like(fwd.k_cmp)
    dv_cmp = np.zeros_like(fwd.v_cmp)
    Cq = plan.offsets["q"]
    Cw = plan.offsets["win"]
    do_c = {c: gs[..., i:i + 1] * dos for i, c in enumerate(("cmp", "slc", "win"))}

    def run(rows_t0, rows_t1, g, kidx_tokens, kmat, vmat, branch):
        qr = _rows(qs, rows_t0, rows_t1, g, h_s)
        dor = _rows(do_c[branch], rows_t0, rows_t1, g, h_s)
        oo, _, pp = dense_attention(qr, kmat, vmat, scale)
        dqr, dkr, dvr = dense_attention_backward(qr, kmat, vmat, pp, oo, dor, scale)
        dq[rows_t0:rows_t1, g * h_s:(g + 1) * h_s] += dqr.reshape(rows_t1 - rows_t0, h_s, d)
        return dkr, dvr

    for Q in range(len(Cq) - 1):
        t0, t1 = int(Cq[Q]), int(Cq[Q + 1])
        b = int(plan.sorted_coords[t0, 0])
        c0, c1 = int(plan.batch_blocks["cmp"][b]), int(plan.batch_blocks["cmp"][b + 1])
        for g in range(h_kv):
            dkr, dvr = run(t0, t1, g, None, fwd.k_cmp[c0:c1, g], fwd.v_cmp[c0:c1, g], "cmp")
            dk_cmp[c0:c1, g] += dkr
            dv_cmp[c0:c1, g] += dvr
            kt = _selected_tokens(plan, fwd.I, Q, g)
            dkr, dvr = run(t0, t1, g, kt, ks[kt, g], vs[kt, g], "slc")
            np.add.at(dk[:, g], kt, dkr)
            np.add.at(dv[:, g], kt, dvr)
    for w in range(len(Cw) - 1):
        t0, t1 = int(Cw[w]), int(Cw[w + 1])
        for g in range(h_kv):
            dkr, dvr = run(t0, t1, g, None, ks[t0:t1, g], vs[t0:t1, g], "win")
            dk[t0:t1, g] += dkr
            dv[t0:t1, g] += dvr
    # mean-pool backward (Eq. 7 with delta = mean, READING R4)
    Cc = plan.offsets["cmp"]
    for j in range(len(Cc) - 1):
        n = Cc[j + 1] - Cc[j]
        dk[Cc[j]:Cc[j + 1]] += dk_cmp[j] / n
        dv[Cc[j]:Cc[j + 1]] += dv_cmp[j] / n
    inv = plan.inv_perm
    return dq[inv], dk[inv], dv[inv], dgates[inv]


# --------------------------------------------------------------------------------------------------
# Per-block gradients for full-size parity (BASELINE configs C3 / C4, where the whole oracle backward
# takes minutes): the same arithmetic as ssa_backward, restricted to the keys of a few blocks. Tested
# equal to ssa_backward on small cases (tests/test_oracle_backward.py), so they inherit its pins
# (central finite differences, closed forms).
# --------------------------------------------------------------------------------------------------
def compression_kv_grad(plan: BlockPlan, q_sorted, k_cmp, v_cmp, gates_sorted, dout_sorted, h_kv: int,
                        scale: float, b: int, cols, chunk: int = 2048, workers: int = 1):
    """dK^cmp, dV^cmp [len(cols), h_kv, d] of the compression branch (Eq. 6 term 1 backward, R15) for the
    compression blocks `cols` (global ids, all in batch item b): the sum over EVERY row (t, h) of item b.
    Rows are processed in chunks of `chunk` (each chunk is dense_attention over all compression keys of
    the item, then dense_attention_backward restricted to the requested key columns — D = <dO_c, O>
    uses the full row); chunk results are summed in chunk order. `workers` > 1 evaluates chunks on a
    thread pool (numpy releases the GIL); the summation order is unchanged."""
    cols = np.asarray(cols, np.int64)
    N, H, d = q_sorted.shape
    h_s = H // h_kv
    t0, t1 = int(plan.batch_tokens[b]), int(plan.batch_tokens[b + 1])
    c0, c1 = int(plan.batch_blocks["cmp"][b]), int(plan.batch_blocks["cmp"][b + 1])
    assert ((cols >= c0) & (cols < c1)).all(), "cols must lie in batch item b"
    loc = cols - c0
    dk = np.zeros((len(cols), h_kv, v_cmp.shape[2]))
    dv = np.zeros((len(cols), h_kv, v_cmp.shape[2]))
    for g in range(h_kv):
        R = _rows(q_sorted, t0, t1, g, h_s)
        DO = _rows(np.asarray(gates_sorted, np.float64)[..., 0:1] * np.asarray(dout_sorted, np.float64),
                   t0, t1, g, h_s)
        Kb = np.asarray(k_cmp[c0:c1, g], np.float64)
        Vb = np.asarray(v_cmp[c0:c1, g], np.float64)

        def one(r0):
            r1 = min(r0 + chunk, R.shape[0])
            o, _, p = dense_attention(R[r0:r1], Kb, Vb, scale)
            _, dkc, dvc = dense_attention_backward(R[r0:r1], Kb[loc], Vb[loc], p[:, loc], o, DO[r0:r1], scale)
            return dkc, dvc

        starts = list(range(0, R.shape[0], chunk))
        if workers > 1:
            from concurrent.futures import ThreadPoolExecutor
            from threadpoolctl import threadpool_limits
            with threadpool_limits(1), ThreadPoolExecutor(workers) as ex:   # no BLAS oversubscription
                parts = list(ex.map(one, starts))
        else:
            parts = [one(r0) for r0 in starts]
        for dkc, dvc in parts:
            dk[:, g] += dkc
            dv[:, g] += dvc
    return dk, dv


def raw_kv_grad_blocks(plan: BlockPlan, q_sorted, k_sorted, v_sorted, gates_sorted, dout_sorted, I, h_kv: int,
                       scale: float, blocks, workers: int = 1) -> dict:
    """{B: (dk, dv) [n_B, h_kv, d]}: gradients of the raw tokens of each selection block B from the
    selection branch (every (Q, g) with B in I[Q, g]: attention over all of Q's selected tokens, Alg. 1 /
    O6) and the window branch (every window holding a token of B, O7) — everything but the compression
    pool share. Each (Q, g) / (window, g) problem is evaluated once for all requested blocks; `workers`
    > 1 evaluates the problems on a thread pool (BLAS single-threaded); contributions are summed in
    problem order."""
    N, H, d = q_sorted.shape
    h_s = H // h_kv
    C = plan.offsets["slc"]
    gs = np.asarray(gates_sorted, np.float64)
    dos = np.asarray(dout_sorted, np.float64)
    do_slc, do_win = gs[..., 1:2] * dos, gs[..., 2:3] * dos          # omega_c dO per branch (Eq. 6)
    want = set(int(B) for B in blocks)
    out = {B: (np.zeros((int(C[B + 1] - C[B]), h_kv, d)), np.zeros((int(C[B + 1] - C[B]), h_kv, v_sorted.shape[2])))
           for B in sorted(want)}
    Cq, Cw = plan.offsets["q"], plan.offsets["win"]
    tasks = []
    for Q in range(len(Cq) - 1):
        for g in range(h_kv):
            hit = sorted(want & set(int(x) for x in I[Q, g]))
            if hit:
                tasks.append(("slc", Q, g, hit))
    wins = sorted(set(int(x) for B in want for x in plan.tok_block["win"][int(C[B]):int(C[B + 1])]))
    for w in wins:
        for g in range(h_kv):
            tasks.append(("win", w, g, None))

    def run(task):
        kind, a, g, hit = task
        if kind == "slc":
            t0, t1 = int(Cq[a]), int(Cq[a + 1])
            kt = _selected_tokens(plan, I, a, g)
            dor = _rows(do_slc, t0, t1, g, h_s)
        else:
            t0, t1 = int(Cw[a]), int(Cw[a + 1])
            kt = np.arange(t0, t1)
            dor = _rows(do_win, t0, t1, g, h_s)
        rows = _rows(q_sorted, t0, t1, g, h_s)
        o, _, p = dense_attention(rows, k_sorted[kt, g], v_sorted[kt, g], scale)
        res = []
        for B in (hit if hit is not None else sorted(want)):
            m = (kt >= C[B]) & (kt < C[B + 1])
            if not m.any():
                continue
            _, dkr, dvr = dense_attention_backward(rows, k_sorted[kt[m], g], v_sorted[kt[m], g], p[:, m], o, dor, scale)
            res.append((B, g, kt[m] - int(C[B]), dkr, dvr))
        return res

    if workers > 1:
        from concurrent.futures import ThreadPoolExecutor
        from threadpoolctl import threadpool_limits
        with threadpool_limits(1), ThreadPoolExecutor(workers) as ex:
            results = list(ex.map(run, tasks))
    else:
        results = [run(t) for t in tasks]
    for res in results:
        for B, g, idx, dkr, dvr in res:
            out[B][0][idx, g] += dkr
            out[B][1][idx, g] += dvr
    return out


def block_kv_grad(plan: BlockPlan, q_sorted, k_sorted, v_sorted, k_cmp, v_cmp, gates_sorted, dout_sorted, I,
                  h_kv: int, scale: float, blocks, workers: int = 1) -> dict:
    """{B: (dk, dv) [n_B, h_kv, d]}: total gradients of the tokens of each selection block B (sorted
    order) = raw-key part (raw_kv_grad_blocks) + the mean-pool share dk^cmp_c / n_c of every compression
    block c inside B (Eq. 7 backward with delta = mean, R4). One compression_kv_grad pass per batch item
    covers all requested blocks of that item."""
    C = plan.offsets["slc"]
    Cc = plan.offsets["cmp"]
    d = q_sorted.shape[2]
    by_item = {}
    for B in blocks:
        by_item.setdefault(int(plan.sorted_coords[int(C[B]), 0]), []).append(int(B))
    out = {}
    for bi, Bs in by_item.items():
        cols = sorted(set(int(x) for B in Bs for x in plan.tok_block["cmp"][int(C[B]):int(C[B + 1])]))
        dkc, dvc = compression_kv_grad(plan, q_sorted, k_cmp, v_cmp, gates_sorted, dout_sorted, h_kv, scale, bi,
                                       np.array(cols, np.int64), workers=workers)
        col_of = {c: i for i, c in enumerate(cols)}
        raw = raw_kv_grad_blocks(plan, q_sorted, k_sorted, v_sorted, gates_sorted, dout_sorted, I, h_kv, scale, Bs,
                                 workers=workers)
        for B in Bs:
            b0, b1 = int(C[B]), int(C[B + 1])
            dk, dv = raw[B]
            for c in sorted(set(int(x) for x in plan.tok_block["cmp"][b0:b1])):
                a, e = int(Cc[c]), int(Cc[c + 1])
                dk[a - b0:e - b0] += dkc[col_of[c]] / (e - a)
                dv[a - b0:e - b0] += dvc[col_of[c]] / (e - a)
            out[B] = (dk, dv)
    return out


# --------------------------------------------------------------------------------------------------
# §8f row 2 — learned compression delta and the gate projection.
# Eq. 7: k^cmp = delta(k + PE(k)), delta = "sparse 3D convolution followed by sparse 3D mean
# pooling" that "compress[es] the entire block". READING R17: the convolution has kernel = stride =
# m_cmp (one output per m_cmp^3 block, one weight matrix per intra-block offset, grouped per kv head),
# evaluated over the ACTIVE tokens only (sparse), and the sparse mean pooling divides by the number of
# active tokens:  k^cmp_B = (1/n_B) sum_{j in B} W[loc(j), g] (k_j + PE[loc(j), g]) + b[g].
# W[loc, g] is a d_out x d_in matrix applied as W @ x. W[loc] = I, b = 0 is the plain mean pool (R4).
# Eq. 6 gates: omega_t = sigmoid(x_t W_g + b_g) — "a linear layer followed by a sigmoid
# activation to the input features" x_t [C]; READING R18: one gate per (head, branch), W_g [C, 3 h_q]
# with column h*3 + c for head h, branch c (cmp, slc, win).
# --------------------------------------------------------------------------------------------------
def compress_learned(plan: BlockPlan, x_sorted, W, b=None, pe=None):
    """x_sorted [N, h_kv, d] -> [N_cmp, h_kv, d_out] (READING R17). W [m^3, h_kv, d_out, d], b [h_kv, d_out]."""
    x = np.asarray(x_sorted, np.float64)
    m = plan.sizes["cmp"]
    loc = local_index(plan.sorted_coords, m)
    if pe is not None:
        x = x + np.asarray(pe, np.float64)[loc]
    W = np.asarray(W, np.float64)
    C = plan.offsets["cmp"]
    out = np.zeros((len(C) - 1, x.shape[1], W.shape[2]))
    for j in range(len(C) - 1):
        for t in range(int(C[j]), int(C[j + 1])):
            for g in range(x.shape[1]):
                out[j, g] += W[loc[t], g] @ x[t, g]
        out[j] /= C[j + 1] - C[j]
    if b is not None:
        out += np.asarray(b, np.float64)[None]
    return out


def compress_learned_backward(plan: BlockPlan, x_sorted, W, dout_cmp, pe=None):
    """Gradients of compress_learned w.r.t. x (sorted order), W and b for the upstream dout_cmp
    [N_cmp, h_kv, d_out] (PE is a constant input)."""
    x = np.asarray(x_sorted, np.float64)
    m = plan.sizes["cmp"]
    loc = local_index(plan.sorted_coords, m)
    if pe is not None:
        x = x + np.asarray(pe, np.float64)[loc]
    W = np.asarray(W, np.float64)
    dy = np.asarray(dout_cmp, np.float64)
    C = plan.offsets["cmp"]
    dx = np.zeros_like(x)
    dW = np.zeros_like(W)
    for j in range(len(C) - 1):
        n = C[j + 1] - C[j]
        for t in range(int(C[j]), int(C[j + 1])):
            for g in range(x.shape[1]):
                dx[t, g] = W[loc[t], g].T @ dy[j, g] / n
                dW[loc[t], g] += np.outer(dy[j, g], x[t, g]) / n
    db = dy.sum(axis=0)
    return dx, dW, db


def gate_projection(x, Wg, bg, h_q: int):
    """omega = sigmoid(x Wg + bg) -> [N, h_q, 3] (READING R18)."""
    z = np.asarray(x, np.float64) @ np.asarray(Wg, np.float64) + np.asarray(bg, np.float64)
    return (1.0 / (1.0 + np.exp(-z))).reshape(len(z), h_q, 3)


def gate_projection_backward(x, Wg, bg, dgates):
    """(dx, dWg, dbg) of gate_projection for the upstream dgates [N, h_q, 3]."""
    x = np.asarray(x, np.float64)
    s = 1.0 / (1.0 + np.exp(-(x @ np.asarray(Wg, np.float64) + np.asarray(bg, np.float64))))
    dz = np.asarray(dgates, np.float64).reshape(len(x), -1) * s * (1.0 - s)
    return dz @ np.asarray(Wg, np.float64).T, x.T @ dz, dz.sum(axis=0)


def ssa_forward_learned(coords, grid, batch, q, k, v, x, *, conv_k, conv_v, gate, h_kv, T, m_cmp, m_slc, m_win,
                        m_q, pe_k=None, pe_v=None, I_override=None):
    """SSA with the learned delta (compress_learned with conv_k = (W_k, b_k), conv_v = (W_v, b_v)) and
    gates from the projection gate = (W_g, b_g) of the input features x [N, C] (original order).
    Returns (ForwardResult, gates [N, H, 3])."""
    q = np.asarray(q, np.float64)
    N, H, d = q.shape
    scale = 1.0 / math.sqrt(d)
    plan = block_build(coords, grid, batch, m_cmp, m_slc, m_win, m_q)
    gates = gate_projection(x, gate[0], gate[1], H)
    P = plan.perm
    qs, ks, vs, gs = q[P], np.asarray(k, np.float64)[P], np.asarray(v, np.float64)[P], gates[P]
    k_cmp = compress_learned(plan, ks, conv_k[0], conv_k[1], pe_k)
    v_cmp = compress_learned(plan, vs, conv_v[0], conv_v[1], pe_v)
    o_c, l_c, probs = compression_attention(plan, qs, k_cmp, v_cmp, h_kv, scale)
    scores = block_scores(plan, probs, h_kv)
    I = topk_all(plan, scores, h_kv, T) if I_override is None else np.asarray(I_override, np.int64)
    o_s, l_s = selection_attention(plan, qs, ks, vs, I, h_kv, scale)
    o_w, l_w = window_attention(plan, qs, ks, vs, h_kv, scale)
    out = gate_combine(o_c, o_s, o_w, gs)
    inv = plan.inv_perm
    f = ForwardResult(out=out[inv], o=dict(cmp=o_c[inv], slc=o_s[inv], win=o_w[inv]),
                      lse=dict(cmp=l_c[inv], slc=l_s[inv], win=l_w[inv]), I=I, scores=scores,
                      k_cmp=k_cmp, v_cmp=v_cmp, plan=plan)
    return f, gates


def ssa_backward_learned(fwd: ForwardResult, q, k, v, x, gates, dout, *, conv_k, conv_v, gate, h_kv,
                         pe_k=None, pe_v=None):
    """Gradients of ssa_forward_learned: (dq, dk, dv, dx, dW_k, db_k, dW_v, db_v, dW_g, db_g), original
    order. Same chain as ssa_backward with the learned delta in place of the mean pool and the gate
    projection after the gates."""
    plan = fwd.plan
    q = np.asarray(q, np.float64)
    N, H, d = q.shape
    h_s = H // h_kv
    scale = 1.0 / math.sqrt(d)
    P = plan.perm
    qs = q[P]
    ks = np.asarray(k, np.float64)[P]
    vs = np.asarray(v, np.float64)[P]
    gs = np.asarray(gates, np.float64)[P]
    dos = np.asarray(dout, np.float64)[P]
    o = {c: fwd.o[c][P] for c in fwd.o}
    dgates = np.stack([(dos * o[c]).sum(axis=2) for c in ("cmp", "slc", "win")], axis=2)
    dq = np.zeros_like(qs)
    dk = np.zeros_like(ks)
    dv = np.zeros_like(vs)
    dk_cmp = np.zeros_like(fwd.k_cmp)
    dv_cmp = np.zeros_like(fwd.v_cmp)
    Cq, Cw = plan.offsets["q"], plan.offsets["win"]
    do_c = {c: gs[..., i:i + 1] * dos for i, c in enumerate(("cmp", "slc", "win"))}

    def run(t0, t1, g, kmat, vmat, branch):
        qr = _rows(qs, t0, t1, g, h_s)
        dor = _rows(do_c[branch], t0, t1, g, h_s)
        oo, _, pp = dense_attention(qr, kmat, vmat, scale)
        dqr, dkr, dvr = dense_attention_backward(qr, kmat, vmat, pp, oo, dor, scale)
        dq[t0:t1, g * h_s:(g + 1) * h_s] += dqr.reshape(t1 - t0, h_s, d)
        return dkr, dvr

    for Q in range(len(Cq) - 1):
        t0, t1 = int(Cq[Q]), int(Cq[Q + 1])
        b = int(plan.sorted_coords[t0, 0])
        c0, c1 = int(plan.batch_blocks["cmp"][b]), int(plan.batch_blocks["cmp"][b + 1])
        for g in range(h_kv):
            dkr, dvr = run(t0, t1, g, fwd.k_cmp[c0:c1, g], fwd.v_cmp[c0:c1, g], "cmp")
            dk_cmp[c0:c1, g] += dkr
            dv_cmp[c0:c1, g] += dvr
            kt = _selected_tokens(plan, fwd.I, Q, g)
            dkr, dvr = run(t0, t1, g, ks[kt, g], vs[kt, g], "slc")
            np.add.at(dk[:, g], kt, dkr)
            np.add.at(dv[:, g], kt, dvr)
    for w in range(len(Cw) - 1):
        t0, t1 = int(Cw[w]), int(Cw[w + 1])
        for g in range(h_kv):
            dkr, dvr = run(t0, t1, g, ks[t0:t1, g], vs[t0:t1, g], "win")
            dk[t0:t1, g] += dkr
            dv[t0:t1, g] += dvr
    dxk, dWk, dbk = compress_learned_backward(plan, ks, conv_k[0], dk_cmp, pe_k)
    dxv, dWv, dbv = compress_learned_backward(plan, vs, conv_v[0], dv_cmp, pe_v)
    dk += dxk
    dv += dxv
    inv = plan.inv_perm
    dx, dWg, dbg = gate_projection_backward(x, gate[0], gate[1], dgates[inv])
    return dq[inv], dk[inv], dv[inv], dx, dWk, dbk, dWv, dbv, dWg, dbg


# --------------------------------------------------------------------------------------------------
# NSA-1D blocking ("treating latent tokens z as a 1D sequence and partitioning it into
# fixed-length blocks based on token indices, analogous to NSA"; the ablation arm of P:394).
# READING R19: block lengths l = m^3 tokens (the token count of the corresponding 3D block), runs of
# consecutive indices per batch item (the last run of an item is shorter), windows non-overlapping.
# --------------------------------------------------------------------------------------------------
def block_offsets_1d(lengths, l: int) -> np.ndarray:
    """C of fixed-length 1D blocks of l tokens over the concatenated batch items (index order)."""
    starts, base = [], 0
    for n in lengths:
        starts += list(range(base, base + int(n), l))
        base += int(n)
    return np.array(starts + [base], dtype=np.int64)


# --------------------------------------------------------------------------------------------------
# SSA with shifted sparse 3D windows (§8f row 3): the window branch of Eq. 6 over the non-overlapping
# m_win^3 windows of the SHIFTED coordinates (x + s, y + s, z + s) — the Swin-style alternation the
# SS-VAE uses for its sparse window attention, applied to SSA's window module;
# compression and selection unchanged. READING R20: s is added to all three axes; windows are formed
# per batch item by floor((coord + s) / m_win).
# --------------------------------------------------------------------------------------------------
def _shifted_windows(coords, m_win: int, shift: int):
    """-> list of ORIGINAL token index arrays, one per non-empty shifted window (python grouping)."""
    groups = {}
    for i, (b, x, y, z) in enumerate(np.asarray(coords).tolist()):
        groups.setdefault((b, (x + shift) // m_win, (y + shift) // m_win, (z + shift) // m_win), []).append(i)
    return [np.array(groups[k], dtype=np.int64) for k in sorted(groups)]


def ssa_forward_shifted(coords, grid, batch, q, k, v, gates, *, shift, h_kv, T, m_cmp, m_slc, m_win, m_q,
                        I_override=None):
    """SSA (Eq. 6) with the window branch on shifted windows. Returns a ForwardResult (original order)
    whose o['win'] / lse['win'] are the shifted-window branch."""
    f = ssa_forward(coords, grid, batch, q, k, v, gates, h_kv=h_kv, T=T, m_cmp=m_cmp, m_slc=m_slc, m_win=m_win,
                    m_q=m_q, I_override=I_override)
    q = np.asarray(q, np.float64)
    N, H, d = q.shape
    h_s = H // h_kv
    scale = 1.0 / math.sqrt(d)
    o_w, l_w = np.zeros((N, H, d)), np.zeros((N, H))
    for t in _shifted_windows(coords, m_win, shift):
        for g in range(h_kv):
            rows = q[t, g * h_s:(g + 1) * h_s].reshape(-1, d)
            oo, ll, _ = dense_attention(rows, np.asarray(k, np.float64)[t, g], np.asarray(v, np.float64)[t, g], scale)
            o_w[t, g * h_s:(g + 1) * h_s] = oo.reshape(len(t), h_s, d)
            l_w[t, g * h_s:(g + 1) * h_s] = ll.reshape(len(t), h_s)
    f.o["win"], f.lse["win"] = o_w, l_w
    f.out = gate_combine(f.o["cmp"], f.o["slc"], o_w, gates)
    return f


def ssa_backward_shifted(fwd: ForwardResult, coords, q, k, v, gates, dout, *, shift, m_win, h_kv):
    """Gradients (dq, dk, dv, dgates) of ssa_forward_shifted (indices constant, R15): the compression
    and selection branches as in ssa_backward (its window term removed by a zero window gate), plus
    the shifted-window branch."""
    g0 = np.asarray(gates, np.float64).copy()
    g0[..., 2] = 0.0
    dq, dk, dv, dg = ssa_backward(fwd, q, k, v, g0, dout, h_kv=h_kv)
    q = np.asarray(q, np.float64)
    N, H, d = q.shape
    h_s = H // h_kv
    scale = 1.0 / math.sqrt(d)
    do = np.asarray(dout, np.float64)
    dg[..., 2] = (do * fwd.o["win"]).sum(axis=2)
    dow = np.asarray(gates, np.float64)[..., 2:3] * do
    for t in _shifted_windows(coords, m_win, shift):
        for g in range(h_kv):
            rows = q[t, g * h_s:(g + 1) * h_s].reshape(-1, d)
            kk, vv = np.asarray(k, np.float64)[t, g], np.asarray(v, np.float64)[t, g]
            oo, _, pp = dense_attention(rows, kk, vv, scale)
            gq, gk, gv = dense_attention_backward(rows, kk, vv, pp, oo, dow[t, g * h_s:(g + 1) * h_s].reshape(-1, d), scale)
            dq[t, g * h_s:(g + 1) * h_s] += gq.reshape(len(t), h_s, d)
            dk[t, g] += gk
            dv[t, g] += gv
    return dq, dk, dv, dg
