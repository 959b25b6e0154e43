"""Probe: PCIe copy throughput alone / concurrent, and overlap with one SSA step (C3)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_17412_b200 import ssa
from ssa_workload import CONFIGS, config_coords, make_inputs

dev = torch.device("cuda:0")
cfg = CONFIGS["C3"]
c, grid, batch = config_coords("C3")
inp = make_inputs(c, grid, batch, 16, 2, 64, "bf16", seed=2)
q, k, v, g, do = (torch.from_numpy(x).to(dev, dtype=torch.bfloat16) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout))
cd = torch.from_numpy(c).to(dev)
acfg = ssa.AttnCfg(h_q=16, h_kv=2, d=64, top_k=8, dtype=torch.bfloat16)
hin = [x.cpu().pin_memory() for x in (q, k, v, g, do)]
din = [torch.empty_like(x) for x in (q, k, v, g, do)]
hout = [torch.empty_like(x, device="cpu").pin_memory() for x in (q, q, k, v, g)]
dout = [torch.empty_like(x) for x in (q, q, k, v, g)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def step():
    plan = ssa.ssa_build_blocks(cd, grid, batch, 4, 8, 8, 8)
    o, saved = ssa.ssa_forward(plan, acfg, q, k, v, g)
    ssa.ssa_backward(plan, acfg, saved, q, k, v, g, do)


def h2d(s):
    with torch.cuda.stream(s):
        for a, b in zip(din, hin):
            a.copy_(b, non_blocking=True)


def d2h(s):
    with torch.cuda.stream(s):
        for a, b in zip(hout, dout):
            a.copy_(b, non_blocking=True)


def wall(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


print("h2d alone ms", wall(lambda: h2d(s1)))
print("d2h alone ms", wall(lambda: d2h(s2)))
print("h2d+d2h concurrent ms", wall(lambda: (h2d(s1), d2h(s2))))
print("step alone ms", wall(step))
print("step + h2d + d2h (no deps) ms", wall(lambda: (h2d(s1), d2h(s2), step())))
print("step + h2d only ms", wall(lambda: (h2d(s1), step())))
print("step + d2h only ms", wall(lambda: (d2h(s2), step())))

# the bench.py e2e pipeline, timed by wall clock and by events
grads = tuple(torch.empty_like(x) for x in (q, k, v, g))
out = torch.empty_like(q)
st = torch.cuda.current_stream()


def stepx(cc, qq, kk, vv, gg, dd, o_, gr_):
    plan = ssa.ssa_build_blocks(cc, grid, batch, 4, 8, 8, 8)
    o, saved = ssa.ssa_forward(plan, acfg, qq, kk, vv, gg, out=o_)
    ssa.ssa_backward(plan, acfg, saved, qq, kk, vv, gg, dd, grads=gr_)


for mode in ("both", "h2d_only", "d2h_only", "none"):
    hin2 = [x.cpu().pin_memory() for x in (cd, q, k, v, g, do)]
    dev_in = [[torch.empty_like(x) for x in (cd, q, k, v, g, do)] for _ in range(2)]
    dev_out = [[torch.empty_like(out)] + [torch.empty_like(x) for x in grads] for _ in range(2)]
    hout2 = [[torch.empty_like(x, device="cpu").pin_memory() for x in dev_out[0]] for _ in range(2)]
    for sl in range(2):
        for a, b in zip(dev_in[sl], (cd, q, k, v, g, do)):
            a.copy_(b)
    n_e = 8
    ev = {key: [torch.cuda.Event() for _ in range(n_e)] for key in ("in", "done", "out")}
    torch.cuda.synchronize()
    t = time.perf_counter()
    stamps = []
    for i in range(n_e):
        slot = i % 2
        with torch.cuda.stream(s1):
            if i >= 2:
                s1.wait_event(ev["done"][i - 2])
            if mode in ("both", "h2d_only"):
                for hx, dx in zip(hin2, dev_in[slot]):
                    dx.copy_(hx, non_blocking=True)
            ev["in"][i].record(s1)
        st.wait_event(ev["in"][i])
        if i >= 2:
            st.wait_event(ev["out"][i - 2])
        cc, qq, kk, vv, gg, dd = dev_in[slot]
        stepx(cc, qq, kk, vv, gg, dd, dev_out[slot][0], tuple(dev_out[slot][1:]))
        ev["done"][i].record(st)
        with torch.cuda.stream(s2):
            s2.wait_event(ev["done"][i])
            if mode in ("both", "d2h_only"):
                for hx, dx in zip(hout2[slot], dev_out[slot]):
                    hx.copy_(dx, non_blocking=True)
            ev["out"][i].record(s2)
        stamps.append(time.perf_counter())
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t) * 1e3
    d = [round((b - a) * 1e3, 1) for a, b in zip(stamps, stamps[1:])]
    print(mode, "ms/step", round(tot / n_e, 2), "cpu iteration gaps", d)
