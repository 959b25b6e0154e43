"""One fwd+bwd step at a given m_q (default 1) and config (default C2) for an ncu launch list:
ncu --metrics gpu__time_duration.sum --csv python tools/mq1_launches.py 1 C3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2505_17412_b200 import ssa
from ssa_workload import config_coords, make_inputs

m_q = int(sys.argv[1]) if len(sys.argv) > 1 else 1
CFG = sys.argv[2] if len(sys.argv) > 2 else "C2"
c, grid, batch = config_coords(CFG)
inp = make_inputs(c, grid, batch, 16, 2, 64, "bf16", seed={"C2": 1, "C3": 2}.get(CFG, 1))
t = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)]
plan = ssa.ssa_build_blocks(torch.from_numpy(c).cuda(), grid, batch, 4, 8, 8, m_q)
acfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=8, dtype=torch.bfloat16, flags=0)
for _ in range(2):
    out, saved = ssa.ssa_forward(plan, acfg, *t[:4])
    ssa.ssa_backward(plan, acfg, saved, *t)
torch.cuda.synchronize()
