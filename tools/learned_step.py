"""One C3 step with the learned delta + gate projection (C = 1024), for ncu launch lists."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_17412_b200 import ssa
from ssa_workload import CONFIGS, config_coords, make_inputs
cfg = CONFIGS["C3"]
c, grid, batch = config_coords("C3")
inp = make_inputs(c, grid, batch, 16, 2, 64, "bf16", seed=2)
dev = torch.device("cuda")
q, k, v, g, do = (torch.from_numpy(x).to(dev, torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout))
C, H, d = 1024, 16, 64
eye = torch.eye(d, device=dev)
W = eye + 0.05 * torch.randn(64, 2, d, d, device=dev)
b0 = torch.zeros(2, d, device=dev)
lcfg = ssa.AttnCfg(h_q=H, h_kv=2, d=d, top_k=8, dtype=torch.bfloat16, learned=ssa.Learned(
    conv_k_w=W, conv_k_b=b0, conv_v_w=W, conv_v_b=b0, x=torch.randn(q.shape[0], C, device=dev).to(torch.bfloat16),
    gate_w=torch.randn(C, 3 * H, device=dev) / math.sqrt(C), gate_b=torch.zeros(3 * H, device=dev)))
cd = torch.from_numpy(c).to(dev)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    plan = ssa.ssa_build_blocks(cd, grid, batch, 4, 8, 8, 8)
    _, sv = ssa.ssa_forward(plan, lcfg, q, k, v, None)
    ssa.ssa_backward(plan, lcfg, sv, q, k, v, None, do)
torch.cuda.synchronize()
print("ok")
