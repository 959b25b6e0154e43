"""One SSA forward+backward on a named config (for ncu captures; not a benchmark)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_17412_b200 import ssa  # noqa: E402
from ssa_workload import CONFIGS, config_coords, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
cfg = CONFIGS[a.config]
c, grid, batch = config_coords(a.config)
inp = make_inputs(c, grid, batch, cfg["H"], cfg["h_kv"], cfg["d"], cfg["dtype"], seed=cfg["seed"])
dt = torch.bfloat16
t = [torch.from_numpy(x).cuda().to(dt) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)]
cd = torch.from_numpy(c).cuda()
acfg = ssa.AttnCfg(h_q=cfg["H"], h_kv=cfg["h_kv"], d=cfg["d"], top_k=cfg["T"], dtype=dt)
for _ in range(a.reps):
    plan = ssa.ssa_build_blocks(cd, grid, batch, cfg["m_cmp"], cfg["m_slc"], cfg["m_win"], cfg["m_q"])
    out, saved = ssa.ssa_forward(plan, acfg, *t[:4])
    ssa.ssa_backward(plan, acfg, saved, *t)
torch.cuda.synchronize()
I = saved.indices().cpu()
import numpy as np  # noqa: E402
u, cnt = np.unique(I.numpy().reshape(-1), return_counts=True)
print("selection popularity: top counts", sorted(cnt)[-10:], "distinct blocks", len(u))
