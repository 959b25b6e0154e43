"""Fixed vs per-tile cost of k_tc_slcwin_fwd: time the forward at C3 for several T and regress the
kernel time on the number of (row-tile pair x key tile) steps. Prints one line per T and the fit."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2505_17412_b200 import ssa
from ssa_workload import make_inputs, sphere_shell, batch_coords

dev = torch.device("cuda", 0)
coords = batch_coords([sphere_shell(128, 58.0, 2.9)])
G = (128, 128, 128)
inp = make_inputs(coords, G, 1, 16, 2, 64, "bf16", seed=2)
q, k, v, g = (torch.from_numpy(x).to(dev, dtype=torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates))
plan = ssa.ssa_build_blocks(torch.from_numpy(coords).to(dev), G, 1, 4, 8, 8, 8)
off_q = plan.offsets(ssa.LEVEL_Q).cpu().numpy().astype(np.int64)
off_s = plan.offsets(ssa.LEVEL_SLC).cpu().numpy().astype(np.int64)
rows = np.diff(off_q) * 8
n_pair = (np.ceil(rows / 128).astype(int) + 1) // 2
res = []
for T in (1, 2, 4, 8, 16, 24):
    cfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=T, dtype=torch.bfloat16)
    for _ in range(3):
        out, saved = ssa.ssa_forward(plan, cfg, q, k, v, g)
    torch.cuda.synchronize()
    ssa.profile_reset(); ssa.profile_enable(True)
    for _ in range(5):
        out, saved = ssa.ssa_forward(plan, cfg, q, k, v, g)
    torch.cuda.synchronize()
    ssa.profile_enable(False)
    t, n = ssa.profile_read("tc_slc_win_fwd")
    ms = t / n
    I = saved.indices().cpu().numpy()
    fill = np.diff(off_s)
    steps = 0
    for Q in range(len(rows)):
        for gi in range(2):
            sel = I[Q, gi][I[Q, gi] >= 0]
            tiles = int(np.ceil(fill[sel] / 128).sum()) + int(np.ceil(fill[Q] / 128))
            steps += n_pair[Q] * tiles
    res.append((T, ms, steps))
    print(f"T={T:3d}  slcwin {ms:.3f} ms  pair-tile steps {steps}  ({ms * 1e3 / steps * 148:.3f} us per step per SM)", flush=True)
A = np.array([[1.0, s] for _, _, s in res])
y = np.array([m for _, m, _ in res])
(a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
print(f"fit: {a:.3f} ms fixed + {b * 1e6:.3f} ns/step  -> per step per SM {b * 1e6 * 148 / 1e3:.3f} us "
      f"(ideal 2 x 128x128 exps at 16/clk/SM, 1.965 GHz = {2 * 128 * 128 / 16 / 1.965e3:.3f} us)")
