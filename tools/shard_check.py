"""Mode-2 data path (ssa_pool + kc_in / kv_event + SSA_LOCAL_ROWS + KV_GRAD_FP32) with virtual ranks on
one GPU at a chosen config, checked against the unsharded run (debug / sanitizer helper).
usage: python tools/shard_check.py [C2|C3] [world]"""
import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2505_17412_b200 import ssa
from paper_2505_17412_b200.shard import shard_ranges
from ssa_workload import CONFIGS, config_coords, make_inputs
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c, grid, batch = config_coords(name)
inp = make_inputs(c, grid, batch, 16, 2, 64, "bf16", seed=11)
dev = torch.device("cuda")
plan = ssa.ssa_build_blocks(torch.from_numpy(c).to(dev), grid, batch, 4, 8, 8, 8)
perm = plan.perm().cpu().numpy()
q, k, v, g, do = [torch.from_numpy(x[perm]).to(dev, dtype=torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)]
base = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=8, dtype=torch.bfloat16, flags=ssa.SSA_INPUT_SORTED)
out0, saved0 = ssa.ssa_forward(plan, base, q, k, v, g)
ref = ssa.ssa_backward(plan, base, saved0, q, k, v, g, do)
torch.cuda.synchronize()
print("unsharded ok", flush=True)
q_rng, tok = shard_ranges(plan, world)
kc = torch.zeros(2, plan.n_blocks[ssa.LEVEL_CMP], 64, device=dev)
vc = torch.zeros_like(kc)
flags = base.flags | ssa.SSA_KV_GRAD_FP32 | ssa.SSA_LOCAL_ROWS
cfgs = [dataclasses.replace(base, flags=flags, q_begin=a, q_end=b) for a, b in q_rng]
for cr, (a, b) in zip(cfgs, tok):
    pk, pv = ssa.ssa_pool(plan, cr, k[a:b].contiguous(), v[a:b].contiguous())
    kc += pk
    vc += pv
torch.cuda.synchronize()
print("pool ok", flush=True)
dk = torch.zeros(k.shape, dtype=torch.float32, device=dev)
for r, (cr, (a, b)) in enumerate(zip(cfgs, tok)):
    ev = torch.cuda.Event()
    ev.record()
    cf = dataclasses.replace(cr, kc_in=kc, vc_in=vc, kv_event=ev)
    o, sv = ssa.ssa_forward(plan, cf, q[a:b].contiguous(), k, v, g[a:b].contiguous())
    torch.cuda.synchronize()
    print("rank", r, "fwd ok", torch.equal(o, out0[a:b]), flush=True)
    gq, gk, gv, gg = ssa.ssa_backward(plan, cr, sv, q[a:b].contiguous(), k, v, g[a:b].contiguous(), do[a:b].contiguous())
    torch.cuda.synchronize()
    print("rank", r, "bwd ok", torch.equal(gq, ref[0][a:b]), torch.equal(gg, ref[3][a:b]), flush=True)
    dk += gk
print("dk rel", float((dk - ref[1].float()).abs().max() / ref[1].float().pow(2).mean().sqrt()))
