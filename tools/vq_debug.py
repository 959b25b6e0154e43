"""Debug helper: the small-query-block parity case at one SSA_VQ_ROWS setting (env), fwd + bwd once,
reporting the first failing launch (run with CUDA_LAUNCH_BLOCKING=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2505_17412_b200 import ssa
from ssa_workload import batch_coords, make_inputs, sphere_shell

m_q = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = batch_coords([sphere_shell(32, 13.0, 2.0)])
inp = make_inputs(c, (32, 32, 32), 1, 16, 2, 64, "bf16", seed=25)
t = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)]
plan = ssa.ssa_build_blocks(torch.from_numpy(c).cuda(), (32, 32, 32), 1, 4, 8, 8, m_q)
acfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=4, dtype=torch.bfloat16, flags=0)
try:
    out, saved = ssa.ssa_forward(plan, acfg, *t[:4])
    torch.cuda.synchronize()
    print("fwd ok", flush=True)
    ssa.ssa_backward(plan, acfg, saved, *t)
    torch.cuda.synchronize()
    print("bwd ok", flush=True)
except Exception as e:  # noqa: BLE001
    print("ERR", str(e)[:300], ssa.lib().ssa_last_error() if hasattr(ssa.lib(), "ssa_last_error") else "")
