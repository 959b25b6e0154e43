"""Helpers for the GPU parity tests: run the CUDA path through the C ABI and the oracle on the same
seeded inputs, and compare with the SURVEY §8c parity protocol."""
from __future__ import annotations

import numpy as np
import torch

import oracle as O
from paper_2505_17412_b200 import ssa


def to_dev(x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype=dtype)


BF16_U = 2.0 ** -8   # unit roundoff of bf16 (p = 8 significand bits): RN error <= 2^-8 |x|, attained just
                     # above a power of two (1.0 -> neighbours 1 - 2^-8, 1 + 2^-7: half-ulp = 2^-8 at 1.0)


def rel_err(x, ref, u=0.0):
    """max(|x - ref| - u |ref|) / rms(ref) — SURVEY §8c parity metric (the north star's "max-abs error
    relative to unit-variance data"). u = 0: undiscounted. u = BF16_U: the round-to-nearest error of a
    bf16-STORED output (its own final rounding, bounded by u |x|) is not charged — every other error is.
    A reference that is analytically zero (rms < 1e-6) is compared in absolute terms."""
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    if not ref.size:
        return 0.0
    rms = float(np.sqrt(np.mean(ref * ref)))
    err = float(np.max(np.maximum(np.abs(x - ref) - u * np.abs(ref), 0.0)))
    return err / rms if rms > 1e-6 else err


# Per-tensor parity report: every comparison made through `record` is kept here and written as JSON at
# the end of the session when SSA_PARITY_REPORT names a file (tests/conftest.py). Each row carries the
# undiscounted error and, for bf16-stored tensors, the error net of the output's own RN rounding.
REPORT = []


def record(test, name, x, ref, tol, stored_bf16=False, **extra):
    """Parity of one tensor (reading R16): fp32-stored tensors must satisfy the undiscounted
    max|x - ref| / rms(ref) <= tol; bf16-stored tensors (out, dq, dk, dv, dgates of the bf16 mode) the
    same with their own final rounding (<= 2^-8 |ref|) not charged. Returns the asserted number."""
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    raw = rel_err(x, ref)
    rn = rel_err(x, ref, BF16_U) if stored_bf16 else raw
    REPORT.append(dict(test=test, tensor=name, n=int(ref.size), stored="bf16" if stored_bf16 else "fp32",
                       max_abs=float(np.max(np.abs(x - ref))) if ref.size else 0.0,
                       rms_ref=float(np.sqrt(np.mean(ref * ref))) if ref.size else 0.0,
                       rel_undiscounted=raw, rel_net_of_output_rounding=rn, tol=tol, ok=bool(rn <= tol), **extra))
    return rn


def internal_to_orig(t_internal: torch.Tensor, perm: np.ndarray):
    """[h_kv][N][h_s][d] (sorted) -> [N][H][d] original order (numpy f64)."""
    hk, n, hs = t_internal.shape[:3]
    x = t_internal.float().cpu().numpy().astype(np.float64)
    x = np.transpose(x, (1, 0, 2) + tuple(range(3, x.ndim)))          # [N][h_kv][h_s](...)
    x = x.reshape((n, hk * hs) + x.shape[3:])
    out = np.empty_like(x)
    out[perm] = x
    return out


def run_gpu(inp, *, h_kv, T, m_cmp, m_slc, m_win, m_q, flags=0, backward=True, pe=None):
    tdt = torch.bfloat16 if inp.dtype == "bf16" else torch.float32
    coords = torch.from_numpy(inp.coords).cuda()
    plan = ssa.ssa_build_blocks(coords, inp.grid, inp.batch, m_cmp, m_slc, m_win, m_q)
    N, H, d = inp.q.shape
    cfg = ssa.AttnCfg(h_q=H, h_kv=h_kv, d=d, top_k=T, dtype=tdt, flags=flags | ssa.SSA_SAVE_SCORES)
    if pe is not None:
        cfg.pe_k, cfg.pe_v = to_dev(pe[0], tdt), to_dev(pe[1], tdt)
    q, k, v, g = (to_dev(x, tdt) for x in (inp.q, inp.k, inp.v, inp.gates))
    out, saved = ssa.ssa_forward(plan, cfg, q, k, v, g)
    res = dict(plan=plan, cfg=cfg, saved=saved, out=out.float().cpu().numpy().astype(np.float64))
    if backward:
        dout = to_dev(inp.dout, tdt)
        dq, dk, dv, dg = ssa.ssa_backward(plan, cfg, saved, q, k, v, g, dout)
        res.update(dq=dq.float().cpu().numpy().astype(np.float64), dk=dk.float().cpu().numpy().astype(np.float64),
                   dv=dv.float().cpu().numpy().astype(np.float64), dgates=dg.float().cpu().numpy().astype(np.float64))
    torch.cuda.synchronize()
    res["I"] = saved.indices().cpu().numpy().astype(np.int64)
    res["scores"] = saved.scores().cpu().numpy()
    res["perm"] = plan.perm().cpu().numpy().astype(np.int64)
    return res


def topk_isolated_check(plan_o, gpu_scores, gpu_I, T):
    """Top-k, isolated: the oracle's top-k on the GPU's fp32 scores must give
    bit-identical index sets, ties included."""
    Cq = plan_o.offsets["q"]
    bad = 0
    for Q in range(len(Cq) - 1):
        b = int(plan_o.sorted_coords[int(Cq[Q]), 0])
        s0, s1 = int(plan_o.batch_blocks["slc"][b]), int(plan_o.batch_blocks["slc"][b + 1])
        for g in range(gpu_I.shape[1]):
            sc = gpu_scores[Q, g, :s1 - s0].astype(np.float64)
            want = O.topk_select(sc, T, base=s0)
            if not np.array_equal(want, gpu_I[Q, g]):
                bad += 1
    return bad


def topk_end_to_end_check(plan_o, oracle_scores, gpu_I, T, delta):
    """Top-k end to end: rows whose f64 relative gap between the T-th and (T+1)-th
    score is < delta are ambiguous (either answer accepted, counted); every other row must match."""
    Cq = plan_o.offsets["q"]
    mismatches, ambiguous = 0, 0
    for (Q, g), sc in oracle_scores.items():
        b = int(plan_o.sorted_coords[int(Cq[Q]), 0])
        s0 = int(plan_o.batch_blocks["slc"][b])
        want = O.topk_select(sc, T, base=s0)
        if np.array_equal(want, gpu_I[Q, g]):
            continue
        srt = np.sort(sc)[::-1]
        if len(srt) > T and (srt[T - 1] - srt[T]) / max(abs(srt[T - 1]), 1e-300) < delta:
            ambiguous += 1
            # the GPU's choice must still be a valid top-T up to the ambiguity band
            got = gpu_I[Q, g]
            got = got[got >= 0] - s0
            assert sc[got].min() >= srt[T - 1] * (1 - 2 * delta)
        else:
            mismatches += 1
    return mismatches, ambiguous
