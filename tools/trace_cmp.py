"""(compression forward trace) Build a traced copy of the library (-DSSA_TRACE), run one backward at C3 and print the KV-outer
pipeline timeline of one CTA (events: 1 producer stage free, 2 MMA issued S^T(j), 3 MMA got P(j),
4 softmax stats ready(j), 5 softmax S ready(j), 6 softmax P buffer free(j), 7 softmax P written(j))."""
import ctypes, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2505_17412_b200 import ssa
from ssa_workload import CONFIGS, config_coords, make_inputs
L = ssa.lib()
f = L.ssa_debug_trace
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
cfg = CONFIGS["C3"]
c, grid, batch = config_coords("C3")
inp = make_inputs(c, grid, batch, 16, 2, 64, "bf16", seed=2)
t = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)]
plan = ssa.ssa_build_blocks(torch.from_numpy(c).cuda(), grid, batch, 4, 8, 8, 8)
acfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=8, dtype=torch.bfloat16)
out, saved = ssa.ssa_forward(plan, acfg, *t[:4])
buf = (ctypes.c_ulonglong * 1024)()
n = f(buf, 768)
ev = np.array(buf[:n], dtype=np.uint64)
clk = (ev >> 16).astype(np.int64)
code = ((ev >> 12) & 0xF).astype(int)
j = (ev & 0xFFF).astype(int)
order = np.argsort(clk)
t0 = clk.min()
names = {1: "P load pass1", 2: "P load pass2", 3: "M issued S (p1)", 4: "M issued S^T (p2)", 5: "M PV wg0",
         6: "M PV wg1", 7: "S p1 S-ready", 8: "S p2 S-ready", 9: "S p1 P-free", 10: "-",
         11: "S p1 P-written"}
print("events", n)
for i in order[:400]:
    print(f"{clk[i]-t0:10d} {names.get(code[i], code[i]):14s} j={j[i]}")
