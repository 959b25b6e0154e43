"""Seeded synthetic inputs for SSA — shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no block partition, no pooling, no attention,
no scoring): it only draws coordinates and feature tensors. It is the one module both the oracle
(`oracle/`) and the CUDA path's tests may use (task rule ③).

Recipe (DESIGN.md §"Input recipe"):
  * geometry: voxel (x,y,z) in [0,G)^3 is active iff | ||(x,y,z)+1/2 - (G/2)*1|| - r | < w/2 — a
    sphere shell, the synthetic stand-in for the paper's active-voxel set of Eq. 1
    ("V = {(x, s(x)) : |s(x)| < tau}") at latent resolution G = R/8.
  * token order: lexicographic (x, y, z) per batch item, batch items concatenated.
  * features: q, k, v, dO ~ N(0,1) from numpy PCG64(seed), drawn in token order; in bf16 mode they
    are rounded to bf16 (round-to-nearest-even) so both sides consume identical values.
  * gates: omega = sigmoid(z), z ~ N(0,1) per (token, head, branch) — post-sigmoid gate values are
    inputs of the boundary ("linear layer followed by a sigmoid").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "sphere_shell", "batch_coords", "round_to_bf16", "SSAInputs", "make_inputs", "CONFIGS",
    "config_coords", "planted_inputs",
]


def sphere_shell(G: int, r: float, w: float) -> np.ndarray:
    """Active voxels of a sphere shell in a G^3 grid, lexicographic (x,y,z) order, int32 [N,3]."""
    ax = np.arange(G, dtype=np.float64) + 0.5 - G / 2.0
    X, Y, Z = np.meshgrid(ax, ax, ax, indexing="ij")
    dist = np.sqrt(X * X + Y * Y + Z * Z)
    mask = np.abs(dist - r) < (w / 2.0)
    idx = np.argwhere(mask)  # argwhere returns lexicographic order for C-ordered arrays
    return idx.astype(np.int32)


def batch_coords(shells: list[np.ndarray]) -> np.ndarray:
    """Concatenate per-shape [n_b,3] coordinate arrays into one int32 [N,4] (b,x,y,z) array."""
    parts = []
    for b, s in enumerate(shells):
        c = np.empty((s.shape[0], 4), dtype=np.int32)
        c[:, 0] = b
        c[:, 1:] = s
        parts.append(c)
    if not parts:
        return np.zeros((0, 4), dtype=np.int32)
    return np.concatenate(parts, axis=0)


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returns float32 holding bf16 values."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) >> 16 << 16
    return (u & 0xFFFFFFFF).astype(np.uint32).view(np.float32).reshape(a.shape)


@dataclass
class SSAInputs:
    coords: np.ndarray          # int32 [N,4] (b,x,y,z)
    grid: tuple                 # (Gx,Gy,Gz)
    batch: int
    q: np.ndarray               # float32 [N,H,d]
    k: np.ndarray               # float32 [N,h_kv,d]
    v: np.ndarray               # float32 [N,h_kv,d]
    gates: np.ndarray           # float32 [N,H,3]  (cmp, slc, win) — Eq. 6 order
    dout: np.ndarray            # float32 [N,H,d]
    dtype: str = "bf16"
    meta: dict = field(default_factory=dict)


def make_inputs(coords: np.ndarray, grid, batch: int, H: int, h_kv: int, d: int,
                dtype: str = "bf16", seed: int = 0) -> SSAInputs:
    """Draw q,k,v,gates,dO for the given coordinates (N(0,1) features, sigmoid(N(0,1)) gates)."""
    N = int(coords.shape[0])
    rng = np.random.Generator(np.random.PCG64(seed))
    q = rng.standard_normal((N, H, d), dtype=np.float32)
    k = rng.standard_normal((N, h_kv, d), dtype=np.float32)
    v = rng.standard_normal((N, h_kv, d), dtype=np.float32)
    z = rng.standard_normal((N, H, 3), dtype=np.float32)
    gates = (1.0 / (1.0 + np.exp(-z.astype(np.float64)))).astype(np.float32)
    dout = rng.standard_normal((N, H, d), dtype=np.float32)
    if dtype == "bf16":
        q, k, v, gates, dout = (round_to_bf16(t) for t in (q, k, v, gates, dout))
    elif dtype != "f32":
        raise ValueError(f"dtype must be 'bf16' or 'f32', got {dtype!r}")
    return SSAInputs(coords=np.ascontiguousarray(coords, dtype=np.int32), grid=tuple(int(g) for g in grid),
                     batch=int(batch), q=q, k=k, v=v, gates=gates, dout=dout, dtype=dtype)


# The five BASELINE.json configs (SURVEY.md §8 "Proposed parameterization", §8d table).
CONFIGS = {
    "C1": dict(shapes=[(32, 13.0, 2.0)], G=32, H=1, h_kv=1, d=64, dtype="f32",
               m_cmp=4, m_slc=4, m_win=4, m_q=4, T=4, seed=0),
    "C2": dict(shapes=[(64, 28.0, 2.5)], G=64, H=16, h_kv=2, d=64, dtype="bf16",
               m_cmp=4, m_slc=8, m_win=8, m_q=8, T=8, seed=1),
    "C3": dict(shapes=[(128, 58.0, 2.9)], G=128, H=16, h_kv=2, d=64, dtype="bf16",
               m_cmp=4, m_slc=8, m_win=8, m_q=8, T=8, seed=2),
    "C4": dict(shapes=[(128, 28.0, 2.0), (128, 36.0, 2.15), (128, 42.0, 2.25), (128, 46.0, 2.45),
                       (128, 50.0, 2.55), (128, 54.0, 2.75), (128, 58.0, 2.85), (128, 60.0, 3.3)],
               G=128, H=16, h_kv=2, d=64, dtype="bf16", m_cmp=4, m_slc=8, m_win=8, m_q=8, T=8, seed=100),
}
CONFIGS["C5"] = dict(CONFIGS["C3"])


def config_coords(name: str, shapes: list | None = None) -> tuple[np.ndarray, tuple, int]:
    """Coordinates, grid and batch size for a named config (or an explicit list of (G,r,w) shells)."""
    cfg = CONFIGS[name]
    shp = cfg["shapes"] if shapes is None else shapes
    shells = [sphere_shell(G, r, w) for (G, r, w) in shp]
    G = cfg["G"]
    return batch_coords(shells), (G, G, G), len(shells)


def planted_inputs(inp: SSAInputs, m_q: int, m_slc: int, T: int, h_s: int, boost: float = 3.0,
                   seed: int = 12345) -> SSAInputs:
    """Planted-selection variant (SURVEY.md §8c parity protocol item 3).

    For every query-block coordinate (b, x//m_q, ...) and kv group g, T random target selection-block
    coordinates (among the occupied ones of the same batch item) are chosen; a shared random unit
    direction u is added (scaled by `boost`) to the q rows of the query block's tokens (all h_s heads of
    g) and to the k rows of the target blocks' tokens. This makes the true top-T gap large, so indices
    must match bit-exactly. Only integer floor division of input coordinates is used here.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    c = inp.coords.astype(np.int64)
    q = inp.q.copy()
    k = inp.k.copy()
    N, H, d = q.shape
    h_kv = k.shape[1]
    for b in range(inp.batch):
        sel = np.nonzero(c[:, 0] == b)[0]
        if sel.size == 0:
            continue
        qkey = [tuple(x) for x in (c[sel, 1:] // m_q)]
        skey = [tuple(x) for x in (c[sel, 1:] // m_slc)]
        sblocks = sorted(set(skey))
        qblocks = sorted(set(qkey))
        s_members: dict = {}
        for i, kk in zip(sel, skey):
            s_members.setdefault(kk, []).append(i)
        q_members: dict = {}
        for i, kk in zip(sel, qkey):
            q_members.setdefault(kk, []).append(i)
        n_sel = min(T, len(sblocks))
        for qb in qblocks:
            for g in range(h_kv):
                picks = rng.choice(len(sblocks), size=n_sel, replace=False)
                u = rng.standard_normal(d)
                u = u / np.linalg.norm(u) * boost * math.sqrt(d)
                qi = np.array(q_members[qb])
                q[qi, g * h_s:(g + 1) * h_s, :] += (u / math.sqrt(d)).astype(np.float32)
                for p in picks:
                    ki = np.array(s_members[sblocks[p]])
                    k[ki, g, :] += (u / math.sqrt(d)).astype(np.float32)
    if inp.dtype == "bf16":
        q, k = round_to_bf16(q), round_to_bf16(k)
    out = SSAInputs(coords=inp.coords, grid=inp.grid, batch=inp.batch, q=q, k=k, v=inp.v,
                    gates=inp.gates, dout=inp.dout, dtype=inp.dtype, meta=dict(inp.meta, planted=True))
    return out
