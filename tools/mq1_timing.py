"""Per-token selection (m_q = 1, the paper's exact Alg. 1 granularity) on the tcgen05 kernels at C2, next
to the query-block path (m_q = m_slc), with the per-kernel split of the per-token step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2505_17412_b200 import ssa
from ssa_workload import CONFIGS, config_coords, make_inputs

CFG = os.environ.get("MQ_CONFIG", "C2")
cfg = CONFIGS[CFG]
c, grid, batch = config_coords(CFG)
inp = make_inputs(c, grid, batch, 16, 2, 64, "bf16", seed={"C2": 1, "C3": 2}.get(CFG, 1))
t = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)]
cc = torch.from_numpy(c).cuda()
for m_q in [int(x) for x in (sys.argv[1:] or ['8', '4', '1'])]:
    plan = ssa.ssa_build_blocks(cc, grid, batch, 4, 8, 8, m_q)
    acfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=8, dtype=torch.bfloat16, flags=0)
    ts = []
    for i in range(13):              # 3 warm-up steps, then the median of 10 (each bracketed by events)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out, saved = ssa.ssa_forward(plan, acfg, *t[:4])
        ssa.ssa_backward(plan, acfg, saved, *t)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"{CFG} m_q={m_q}: {ts[len(ts) // 2]:.2f} ms fwd+bwd (median of 10; {'tcgen05' if saved.used_tcgen05 else 'SIMT'}), "
          f"bwd ws {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB peak, N={c.shape[0]}", flush=True)
    ssa.profile_reset()
    ssa.profile_enable(True)
    out, saved = ssa.ssa_forward(plan, acfg, *t[:4])
    ssa.ssa_backward(plan, acfg, saved, *t)
    torch.cuda.synchronize()
    ssa.profile_enable(False)
    print("   ", {kn: round(ssa.profile_read(kn)[0], 3) for kn in ("tc_cmp_fwd", "tc_slc_win_fwd", "tc_bwd_dq", "tc_bwd_kv", "tc_bwd_cmp_kv")}, flush=True)

# per-kernel split of the per-token (SIMT) step
ssa.profile_reset()
ssa.profile_enable(True)
out, saved = ssa.ssa_forward(plan, acfg, *t[:4])
ssa.ssa_backward(plan, acfg, saved, *t)
torch.cuda.synchronize()
ssa.profile_enable(False)
for kn in ("tc_cmp_fwd", "tc_slc_win_fwd", "tc_bwd_dq", "tc_bwd_kv", "tc_bwd_cmp_kv",
           "k_cmp_fwd", "k_attn_fwd(slc)", "k_attn_fwd(win)", "k_dq", "k_slc_dkdv", "k_win_bwd", "k_cmp_dkdv"):
    ms, n = ssa.profile_read(kn)
    if n:
        print(f"  {kn}: {ms:.2f} ms")
