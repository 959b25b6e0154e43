"""Timeline of one CTA (blockIdx (5, 0)) of a traced kernel at C3: run with SSA_LIB pointing at a library built
with -DSSA_TRACE. `python tools/trace_cmp.py` = compression forward, `... dq` = dQ backward kernel."""
import ctypes, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2505_17412_b200 import ssa
from ssa_workload import CONFIGS, config_coords, make_inputs
L = ssa.lib()
which = sys.argv[1] if len(sys.argv) > 1 else "cmp"
f = {"cmp": L.ssa_debug_trace, "dq": L.ssa_debug_trace_dq, "kv": L.ssa_debug_trace_kv, "sw": L.ssa_debug_trace_sw}[which]
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
cfg = CONFIGS["C3"]
c, grid, batch = config_coords("C3")
inp = make_inputs(c, grid, batch, 16, 2, 64, "bf16", seed=2)
t = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)]
plan = ssa.ssa_build_blocks(torch.from_numpy(c).cuda(), grid, batch, 4, 8, 8, 8)
acfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=8, dtype=torch.bfloat16)
out, saved = ssa.ssa_forward(plan, acfg, *t[:4])
if which in ("dq", "kv"):
    ssa.ssa_backward(plan, acfg, saved, *t)
buf = (ctypes.c_ulonglong * 2048)()
n = f(buf, 1536)
ev = np.array(buf[:n], dtype=np.uint64)
clk = (ev >> 16).astype(np.int64)
code = ((ev >> 12) & 0xF).astype(int)
j = (ev & 0xFFF).astype(int)
order = np.argsort(clk)
t0 = clk.min()
names = {1: "P load pass1", 2: "P load pass2", 3: "M issued S (p1)", 4: "M issued S^T (p2)", 5: "M PV wg0",
         6: "M PV wg1", 7: "S p1 S-ready", 8: "S p2 S-ready", 9: "S p1 P-free", 10: "-",
         11: "S p1 P-written"}
if which == "dq":
    names = {1: "P load", 3: "M issued S", 5: "M dQ issued", 7: "S S-ready", 8: "S turn-in", 9: "S turn-out",
             10: "S dS-free", 11: "S dS-written"}
if which == "kv":
    names = {1: "P row tile", 3: "M S^T issued", 5: "M dVdK issued", 7: "S S-ready", 8: "S turn-in", 9: "S turn-out",
             11: "S P written"}
if which == "sw":
    names = {0: "S epi staged", 2: "S epi batch0", 4: "S epi batch1", 1: "P Q load", 3: "M S issued", 5: "M PV issued", 6: "S wait S", 7: "S S-ready", 8: "S turn-wait",
             9: "S turn-in", 10: "S turn-out", 11: "S S-loaded", 12: "S p_free", 13: "S epi wait O", 14: "S epi O-ready", 15: "S epi done"}
print("events", n)
for i in order[:1600]:
    print(f"{clk[i]-t0:10d} {names.get(code[i], code[i]):14s} j={j[i]}")
