"""Per-token selection: the per-block selection pass (default) against the union-masked virtual level
(SSA_VQ_BLOCKSEL=0) on the same inputs — saved O_slc / LSE_slc and out, max differences."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2505_17412_b200 import ssa
from ssa_workload import config_coords, make_inputs

cfgn = sys.argv[1] if len(sys.argv) > 1 else "C2"
c, grid, batch = config_coords(cfgn)
inp = make_inputs(c, grid, batch, 16, 2, 64, "bf16", seed=1)
t = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates)]
plan = ssa.ssa_build_blocks(torch.from_numpy(c).cuda(), grid, batch, 4, 8, 8, 1)
acfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=8, dtype=torch.bfloat16)
res = {}
for mode in ("1", "0"):
    os.environ["SSA_VQ_BLOCKSEL"] = mode
    out, saved = ssa.ssa_forward(plan, acfg, *t)
    torch.cuda.synchronize()
    o1, l1 = saved.branch(1)
    res[mode] = (out.float().clone(), o1.float().clone(), l1.float().clone())
print({k: v for k, v in zip(("out_maxdiff",), [float((res["1"][0] - res["0"][0]).abs().max())])})
print("o_slc maxdiff", float((res["1"][1] - res["0"][1]).abs().max()), "lse_slc maxdiff",
      float((res["1"][2] - res["0"][2]).abs().max()), "o_slc rms", float(res["0"][1].pow(2).mean().sqrt()))
