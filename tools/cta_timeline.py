"""Per-CTA timeline of k_tc_slcwin_fwd at C3 (library built with -DSSA_TRACE, SSA_LIB pointing at it):
kernel span, SM busy fraction, tail, and the fit CTA duration = a + b * (row-tile pairs x key tiles)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2505_17412_b200 import ssa
from ssa_workload import config_coords, make_inputs
L = ssa.lib()
f = L.ssa_debug_cta_stamps
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
c, grid, batch = config_coords("C3")
inp = make_inputs(c, grid, batch, 16, 2, 64, "bf16", seed=2)
t = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates)]
plan = ssa.ssa_build_blocks(torch.from_numpy(c).cuda(), grid, batch, 4, 8, 8, 8)
acfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=int(sys.argv[1]) if len(sys.argv) > 1 else 8, dtype=torch.bfloat16)
for _ in range(3):
    out, saved = ssa.ssa_forward(plan, acfg, *t)
torch.cuda.synchronize()
nq = plan.offsets(ssa.LEVEL_Q).numel() - 1
n = 2 * nq
buf = (ctypes.c_ulonglong * (3 * n))()
f(buf, n)
a = np.array(buf[:], dtype=np.int64).reshape(n, 3)
st, en, sm = a[:, 0], a[:, 1], a[:, 2]
t0 = st.min()
span = en.max() - t0
dur = en - st
print(f"CTAs {n}  span {span / 1e3:.1f} us  sum(dur)/(148*span) {dur.sum() / (148 * span):.3f}  "
      f"mean dur {dur.mean() / 1e3:.1f} us  min {dur.min() / 1e3:.1f} max {dur.max() / 1e3:.1f}")
last_start = np.sort([en[sm == s].max() for s in np.unique(sm)])
print(f"SM finish times (us): first {(last_start[0] - t0) / 1e3:.1f}  median {(np.median(last_start) - t0) / 1e3:.1f}  last {(last_start[-1] - t0) / 1e3:.1f}")
gaps = []
for s in np.unique(sm):
    idx = np.argsort(st[sm == s])
    ss, ee = st[sm == s][idx], en[sm == s][idx]
    gaps += list(ss[1:] - ee[:-1])
print(f"gap between consecutive CTAs on an SM: mean {np.mean(gaps) / 1e3:.2f} us, median {np.median(gaps) / 1e3:.2f} us")
# work per CTA
off_q = plan.offsets(ssa.LEVEL_Q).cpu().numpy().astype(np.int64)
off_s = plan.offsets(ssa.LEVEL_SLC).cpu().numpy().astype(np.int64)
fill = np.diff(off_s)
I = saved.indices().cpu().numpy()
qo = np.arange(nq)   # blockIdx.x -> Q = q_order[x]; recover by matching rows is not needed for the fit:
# CTA (x, y) processes Q = q_order[x]; q_order is not exported, so fit on the per-Q work sorted like durations
work = []
pairs = []
for Q in range(nq):
    rows = (off_q[Q + 1] - off_q[Q]) * 8
    npair = (int(np.ceil(rows / 128)) + 1) // 2
    for gi in range(2):
        sel = I[Q, gi][I[Q, gi] >= 0]
        tiles = int(np.ceil(fill[sel] / 128).sum()) + int(np.ceil(fill[Q] / 128))
        work.append(npair * tiles)
        pairs.append(npair)
w = np.sort(np.array(work))
d = np.sort(dur)
A = np.stack([np.ones_like(w, dtype=float), w.astype(float)], 1)
(c0, c1), *_ = np.linalg.lstsq(A, d.astype(float), rcond=None)
print(f"rank-matched fit: CTA duration = {c0 / 1e3:.2f} us + {c1:.1f} ns x pair-tile steps  "
      f"(ideal per step {2 * 128 * 128 / 16 / 1.965:.0f} ns)")
