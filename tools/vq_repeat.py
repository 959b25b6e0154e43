"""Debug helper: repeat the m_q small-query-block fwd+bwd N times in one process (env as given)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2505_17412_b200 import ssa
from ssa_workload import batch_coords, make_inputs, sphere_shell

m_q, n = int(sys.argv[1]), int(sys.argv[2])
c = batch_coords([sphere_shell(32, 13.0, 2.0)])
inp = make_inputs(c, (32, 32, 32), 1, 16, 2, 64, "bf16", seed=25)
t = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)]
cc = torch.from_numpy(c).cuda()
for i in range(n):
    junk = torch.full((int(2e8),), float("nan"), device="cuda")   # stale NaN garbage in the allocator
    del junk
    plan = ssa.ssa_build_blocks(cc, (32, 32, 32), 1, 4, 8, 8, m_q)
    acfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=4, dtype=torch.bfloat16, flags=0)
    out, saved = ssa.ssa_forward(plan, acfg, *t[:4])
    dq, dk, dv, dg = ssa.ssa_backward(plan, acfg, saved, *t)
    torch.cuda.synchronize()
    print(i, "ok", float(dk.float().abs().sum()), float(dq.float().abs().sum()), flush=True)
