"""Small SSA forward+backward on every path, for compute-sanitizer (memcheck / racecheck / synccheck):
0 tcgen05, 1 window-only, 2 SIMT bf16, 3 SIMT fp32, 4 learned delta + gate projection (tcgen05),
5 shifted-window SSA (SSA_NO_WINDOW + SSA_WINDOW_ONLY | SSA_ACCUMULATE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2505_17412_b200 import ssa
from ssa_workload import make_inputs, sphere_shell, batch_coords
c = batch_coords([sphere_shell(24, 9.0, 2.0), sphere_shell(24, 6.0, 2.0)])
CASES = ((torch.bfloat16, 0), (torch.bfloat16, ssa.SSA_WINDOW_ONLY), (torch.bfloat16, ssa.SSA_FORCE_SIMT),
         (torch.float32, 0), (torch.bfloat16, "learned"), (torch.bfloat16, "shifted"))
only = [int(a) for a in sys.argv[1:]] or range(len(CASES))
for dt, flags in (CASES[i] for i in only):
    inp = make_inputs(c, (24, 24, 24), 2, 8, 2, 64, "bf16" if dt == torch.bfloat16 else "f32", seed=3)
    cd = torch.from_numpy(c).cuda()
    t = [torch.from_numpy(x).cuda().to(dt) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)]
    if flags == "shifted":
        cfg = ssa.AttnCfg(h_q=8, h_kv=2, d=64, top_k=4, dtype=dt)
        out, ctx = ssa.shifted_window_ssa(cd, (24, 24, 24), 2, 4, 8, 4, cfg, *t[:4])
        g = ssa.shifted_window_ssa_backward(ctx, *t)
        saved = ctx[4]
    else:
        learned = None
        if flags == "learned":
            eye = torch.eye(64, device="cuda").expand(64, 2, 64, 64).contiguous()
            learned = ssa.Learned(conv_k_w=eye, conv_k_b=torch.zeros(2, 64, device="cuda"), conv_v_w=eye,
                                  conv_v_b=torch.zeros(2, 64, device="cuda"),
                                  x=torch.randn(len(c), 96, device="cuda").to(dt),
                                  gate_w=torch.randn(96, 24, device="cuda") / 10, gate_b=torch.zeros(24, device="cuda"))
        plan = ssa.ssa_build_blocks(cd, (24, 24, 24), 2, 4, 8, 8, 8)
        cfg = ssa.AttnCfg(h_q=8, h_kv=2, d=64, top_k=4, dtype=dt, flags=0 if learned else flags, learned=learned)
        out, saved = ssa.ssa_forward(plan, cfg, *t[:4])
        g = ssa.ssa_backward(plan, cfg, saved, *t)
    torch.cuda.synchronize()
    print(dt, flags, "tc" if saved.used_tcgen05 else "simt", float(out.float().abs().sum()), float(g[0].float().abs().sum()),
          flush=True)
