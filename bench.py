#!/usr/bin/env python
"""bench.py — SSA forward+backward at 1024^3-resolution token counts (BASELINE.json configs[2], "C3").

One step = the whole hot path of SURVEY §8(a) on one batch of synthetic input: block build (a1),
permute (a2), pool (a3), compression attention + Eq. 8 scores + top-k (a4, a5), selection + window
attention (a6, a7), gated sum (a8) and the backward (a9), all in libssa_b200's kernels.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU): weak scaling — every rank processes its own shape(s); no
collective on the data path (SSA has no parameters; shapes are independent, SURVEY §8e mode 1).
Only the timing barrier and the max-over-ranks reduction use torch.distributed.

Prints ONE JSON line on rank 0. `value` = whole-job ms per shape (fwd+bwd) = max-over-ranks step
time / shapes processed per step by all ranks (lower is better).
"""
from __future__ import annotations

import argparse
import json
import re
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SSA fwd+bwd ms & tensor-pipe % at 1024^3 tokens; speedup vs full attention"
UNIT = "ms/shape (fwd+bwd, 1024^3-res shape)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-full", action="store_true", help="skip the full-attention comparator")
    ap.add_argument("--no-window", action="store_true", help="skip the window-only (SSA_WINDOW_ONLY) context timing")
    ap.add_argument("--no-learned", action="store_true", help="skip the learned-delta / gate-projection context timing")
    ap.add_argument("--force-simt", action="store_true")
    ap.add_argument("--exchange", default="allgather", choices=["allgather", "fetch"],
                    help="C5 / hybrid K/V exchange: bulk all-gather or one-sided fetch of the selected blocks")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: validate the N>1 logic with several ranks on one GPU)")
    ap.add_argument("--cpu-sample", type=int, default=0, help="query blocks in the oracle sample (0: 4 per core)")
    ap.add_argument("--cpu-check-c2", type=int, default=1, help="also run the oracle on all of C2 (extrapolation check)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING recipe)."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return

        def rd():
            for line in self.proc.stdout:
                self.rows.append([x.strip() for x in line.split(",")])
        self.thread = threading.Thread(target=rd, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for n, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def workload(config: str, rank: int, world: int):
    """Shapes of this rank. C3: one 1024^3-res shell per rank (weak scaling); C5: the same shell on every
    rank, its query blocks sharded (strong scaling); C4: the whole 8-shape batch (N > 1: placed by
    shard.hybrid_plan, see hybrid_step)."""
    from ssa_workload import CONFIGS, batch_coords, sphere_shell
    cfg = CONFIGS[config]
    shells = [sphere_shell(*s) for s in cfg["shapes"]]
    return cfg, batch_coords(shells), (cfg["G"],) * 3, len(shells)


def hybrid_step(ssa, torch, dist, dev, cfg, acfg, rank, world, exchange="allgather"):
    """C4 on N > 1 ranks (SURVEY §8e hybrid, shard.HybridBatch): the batch's query blocks on one cost line
    cut into N equal pieces; shapes a rank holds entirely run whole as one batch plan (mode 1, no
    collective), shapes cut by a piece boundary run ssa_step_sharded over their sub-group (mode 2).
    Every rank holds the batch's inputs (identical seeds per shape); a step includes every block build
    and the gather of the rank's own rows. Returns (step, info)."""
    from paper_2505_17412_b200.shard import HybridBatch
    from ssa_workload import batch_coords, make_inputs, sphere_shell
    G = (cfg["G"],) * 3
    ms = (cfg["m_cmp"], cfg["m_slc"], cfg["m_win"], cfg["m_q"])
    coords = [batch_coords([sphere_shell(*sh)]) for sh in cfg["shapes"]]
    tens = []
    for s, c in enumerate(coords):
        inp = make_inputs(c, G, 1, cfg["H"], cfg["h_kv"], cfg["d"], cfg["dtype"], seed=cfg["seed"] + s)
        tens.append([torch.from_numpy(x).to(dev, dtype=acfg.dtype) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout)])
    hb = HybridBatch(coords, G, ms, acfg, rank, world, dev, exchange=exchange)
    info = {"whole_shapes": hb.whole, "split_shapes": [(s, list(g)) for s, g in hb.split],
            "plan": [[(s, a, b, len(g)) for (s, a, b, g) in items] for items in hb.plan]}

    def step():
        hb.step(tens)
        return None, None
    return step, info


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    import torch
    import torch.distributed as dist
    local = local % max(1, torch.cuda.device_count())    # gloo validation runs: several ranks per GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    from paper_2505_17412_b200 import ssa
    from ssa_workload import make_inputs

    cfg, coords, grid, batch = workload(args.config, rank, world)
    H, h_kv, d, T = cfg["H"], cfg["h_kv"], cfg["d"], cfg["T"]
    ms = (cfg["m_cmp"], cfg["m_slc"], cfg["m_win"], cfg["m_q"])
    tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    inp = make_inputs(coords, grid, batch, H, h_kv, d, cfg["dtype"], seed=cfg["seed"] + rank)
    N = coords.shape[0]
    # inputs resident in HBM before the timed region
    c_d = torch.from_numpy(coords).to(dev)
    q, k, v, g, do = (torch.from_numpy(x).to(dev, dtype=tdt) for x in (inp.q, inp.k, inp.v, inp.gates, inp.dout))
    flags = ssa.SSA_FORCE_SIMT if args.force_simt else 0
    acfg = ssa.AttnCfg(h_q=H, h_kv=h_kv, d=d, top_k=T, dtype=tdt, flags=flags)
    grads = tuple(torch.empty_like(x) for x in (q, k, v, g))
    out = torch.empty_like(q)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    st = torch.cuda.current_stream(dev)

    sharded = args.config == "C5"
    hybrid = args.config == "C4" and world > 1
    hybrid_info = None
    comm = torch.cuda.Stream(dev)
    if hybrid:
        hstep, hybrid_info = hybrid_step(ssa, torch, dist, dev, cfg, acfg, rank, world, exchange=args.exchange)

    def step(qq=q, kk=k, vv=v, gg=g, dd=do, o_=out, gr_=grads, cc=c_d, after_build=None):
        if hybrid:
            return hstep()
        plan = ssa.ssa_build_blocks(cc, grid, batch, *ms)
        if after_build is not None:
            after_build()
        if sharded:
            # one shape, query blocks sharded over the ranks (SURVEY §8e mode 2): every rank builds the
            # same plan and gathers its own rows (plan order); pooled-key all-reduce, K/V all-gather
            # overlapped with the compression branch, dK/dV reduce-scatter (shard.ssa_step_sharded)
            from paper_2505_17412_b200.shard import shard_ranges, ssa_step_sharded
            _, tok = shard_ranges(plan, world)
            a, b = tok[rank]
            rows = plan.perm()[a:b].long()
            loc = [x[rows] for x in (qq, kk, vv, gg, dd)]
            ssa_step_sharded(plan, acfg, *loc, rank=rank, world=world, comm_stream=comm, exchange=args.exchange)
            return plan, None
        o, saved = ssa.ssa_forward(plan, acfg, qq, kk, vv, gg, out=o_)
        ssa.ssa_backward(plan, acfg, saved, qq, kk, vv, gg, dd, grads=gr_)
        return plan, saved

    for _ in range(max(args.warmup, 3) if args.warmup > 0 else 3):
        plan, saved = step()
    torch.cuda.synchronize(dev)
    if saved is None:     # sharded / hybrid: one unsharded forward of the batch for the work accounting below
        plan = ssa.ssa_build_blocks(c_d, grid, batch, *ms)
        saved = ssa.ssa_forward(plan, acfg, q, k, v, g, out=out)[1]
        torch.cuda.synchronize(dev)
    used_tc = saved.used_tcgen05

    # ---- timed region: K steps, L2 flushed between steps (outside the events) ----
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    ssa.reset_launch_count()
    ssa.profile_reset()
    ssa.profile_enable(True)
    times = []
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        step()
        e1.record(st)
        times.append((e0, e1))
    torch.cuda.synchronize(dev)
    ssa.profile_enable(False)
    launches = ssa.launch_count()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in times]
    total_ms = float(sum(step_ms))
    kernel_names = ["tc_cmp_fwd", "tc_slc_win_fwd", "tc_bwd_dq", "tc_bwd_kv", "tc_bwd_cmp_kv",
                    "k_cmp_fwd", "k_attn_fwd(slc)", "k_attn_fwd(win)", "k_dq", "k_slc_dkdv", "k_win_bwd", "k_cmp_dkdv"]
    ktimes = {}
    for kn in kernel_names:
        t, n = ssa.profile_read(kn)
        if n:
            ktimes[kn] = (t, n)
    ssa.profile_reset()
    from paper_2505_17412_b200.shard import max_over_ranks
    total_ms = max_over_ranks(total_ms, dev)
    ms_per_step = total_ms / args.steps
    shapes_per_step = batch * (1 if (sharded or hybrid) else world)
    value = ms_per_step / shapes_per_step

    # ---- algorithmic work of the dominant kernel ----
    I = saved.indices().cpu().numpy()
    off_slc = plan.offsets(ssa.LEVEL_SLC).cpu().numpy()
    off_q = plan.offsets(ssa.LEVEL_Q).cpu().numpy()
    off_w = plan.offsets(ssa.LEVEL_WIN).cpu().numpy()
    bb_c = plan.batch_blocks(ssa.LEVEL_CMP).cpu().numpy()
    bt = np.searchsorted(coords[np.argsort(coords[:, 0], kind="stable"), 0], np.arange(batch + 1))
    h_s = H // h_kv
    n_cmp_b = np.diff(bb_c)
    ntok_b = np.diff(bt)
    E_cmp = float(np.sum(ntok_b * n_cmp_b)) * H
    fill = np.diff(off_slc)
    qn = np.diff(off_q)
    E_slc = float(sum(qn[Q] * h_s * fill[I[Q, gi][I[Q, gi] >= 0]].sum() for Q in range(len(qn)) for gi in range(h_kv)))
    E_win = float(np.sum(np.diff(off_w).astype(np.float64) ** 2)) * H
    # Per-kernel ALGORITHMIC work, SURVEY §8(d) / DESIGN.md §5 (2 flops per MAC, E = score elements):
    #   forward: 4d per element (QK^T, PV) + 2d for the a4 score pass (Eq. 8 needs S a second time
    #            after the LSE is known), exponentials: 1 per element, 2 for a4 (LSE pass + Eq. 8 pass);
    #   backward: 10d per element (FA convention: S, dP, dQ, dK, dV once). Our backward computes S and dP
    #            in both the Q-outer (dQ) and the KV-outer (dK, dV) kernel, so the algorithmic 10d is
    #            split 6d (S, dP, dQ) to tc_bwd_dq and 4d (dK, dV) to the KV-outer kernels; the 4d they
    #            recompute is reported separately as "executed" work, not credited to the roofline.
    E_sw = E_slc + E_win
    models = {   # kernel: (algorithmic flops, algorithmic exps, executed flops)
        "tc_cmp_fwd": (6 * d * E_cmp, 2 * E_cmp, 8 * d * E_cmp),      # executed: S twice in hi + lo (K^cmp split)
        "tc_slc_win_fwd": (4 * d * E_sw, E_sw, 4 * d * E_sw),
        "tc_bwd_dq": (6 * d * (E_cmp + E_sw), E_cmp + E_sw, 6 * d * (E_cmp + E_sw)),
        "tc_bwd_kv": (4 * d * E_sw, 0.0, 8 * d * E_sw),
        "tc_bwd_cmp_kv": (4 * d * E_cmp, 0.0, 8 * d * E_cmp),
    }
    peaks, peak_src = load_peaks()
    roofline = None
    cands = [k for k in models if k in ktimes]
    if cands:
        dom = max(cands, key=lambda k: ktimes[k][0] / ktimes[k][1])
        t, n = ktimes[dom]
        avg_s = t / n / 1e3
        flops, exps, _ = models[dom]
        mhz = float(peaks.get("sm_max_mhz", 1965.0))
        tc_peak = float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))          # TFLOP/s (fp16 = bf16 rate)
        xu_peak = 148 * 16 * mhz * 1e6 / 1e12                                              # T ex2/s: 16 MUFU.EX2/clk/SM
        tc_ach, xu_ach = flops / avg_s / 1e12, exps / avg_s / 1e12
        traffic = None
        import glob
        for tf in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_traffic_*.json")))[-1:]:
            tj = json.load(open(tf))
            ncu_name = {"tc_cmp_fwd": "k_tc_cmp_fwd", "tc_slc_win_fwd": "k_tc_slcwin_fwd", "tc_bwd_dq": "k_tc_dq",
                        "tc_bwd_kv": "k_tc_dkdv", "tc_bwd_cmp_kv": "k_tc_dkdv#1"}[dom]   # dkdv: raw launch, then cmp
            for kname, val in tj.items():
                if re.sub(r"<[^<>]*>", "", kname).endswith(ncu_name):   # template arguments dropped
                    traffic = {"dram_bytes_per_launch": val, "source": os.path.relpath(tf, ROOT)}
        if xu_ach / xu_peak >= tc_ach / tc_peak:
            roofline = {"kernel": dom, "bound": "alu", "achieved": round(xu_ach, 4), "peak": round(xu_peak, 4),
                        "unit": "Tex2/s", "frac": round(xu_ach / xu_peak, 4),
                        "peak_source": "MUFU.EX2 16/clk/SM (guide unit count) x 148 SMs x sm_max_mhz (" + peak_src + "); "
                                       "measured on this B200: 15.8/clk/SM at full occupancy (tools/xu_microbench.cu, "
                                       "DESIGN.md §5)",
                        "frac_vs_measured_mufu": round(xu_ach / (xu_peak * 15.8 / 16), 4)}
        else:
            roofline = {"kernel": dom, "bound": "tensor", "achieved": round(tc_ach, 2), "peak": round(tc_peak, 1),
                        "unit": "TFLOP/s", "frac": round(tc_ach / tc_peak, 4),
                        "peak_source": peak_src + " bf16_tflops_sustained"}
        roofline.update({"traffic": traffic, "tensor_view": {"achieved_tflops": round(tc_ach, 2), "peak": round(tc_peak, 1),
                                                             "frac": round(tc_ach / tc_peak, 4)},
                         "mufu_view": {"achieved_tex2": round(xu_ach, 4), "peak": round(xu_peak, 4),
                                       "frac": round(xu_ach / xu_peak, 4)},
                         "algorithmic_flops_per_launch": flops, "exp2_per_launch": exps,
                         "avg_launch_ms": round(t / n, 4), "share_of_step": round(t / n / ms_per_step, 4)})
    if hybrid:      # a rank's kernels cover only its share of the batch: no per-kernel roofline at N > 1
        roofline, cands = None, []
    kernel_ms = {kn: round(t / n, 4) for kn, (t, n) in ktimes.items()}
    # every tensor-core kernel against both of its units (same algorithmic work model as the roofline);
    # "selected-block attention" (north star: >= 50% of dense bf16 peak) = tc_slc_win_fwd forward and
    # tc_bwd_kv backward (selection + window keys)
    kernel_roofline = {}
    if cands:
        mhz = float(peaks.get("sm_max_mhz", 1965.0))
        tc_peak = float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
        xu_peak = 148 * 16 * mhz * 1e6 / 1e12
        for kn in cands:
            t, n = ktimes[kn]
            avg_s = t / n / 1e3
            flops, exps, xflops = models[kn]
            kernel_roofline[kn] = {"tflops": round(flops / avg_s / 1e12, 1), "tensor_frac": round(flops / avg_s / 1e12 / tc_peak, 4),
                                   "tex2_per_s": round(exps / avg_s / 1e12, 3), "mufu_frac": round(exps / avg_s / 1e12 / xu_peak, 4),
                                   "executed_tflops": round(xflops / avg_s / 1e12, 1)}
        # step level: forward 4d ΣE + 2d E_cmp, backward 10d ΣE
        fw = [kn for kn in ("tc_cmp_fwd", "tc_slc_win_fwd") if kn in ktimes]
        bw = [kn for kn in ("tc_bwd_dq", "tc_bwd_kv", "tc_bwd_cmp_kv") if kn in ktimes]
        if fw and bw:
            t_f = sum(ktimes[kn][0] / ktimes[kn][1] for kn in fw) / 1e3
            t_b = sum(ktimes[kn][0] / ktimes[kn][1] for kn in bw) / 1e3
            E_all = E_cmp + E_sw
            kernel_roofline["forward_kernels"] = {"tflops": round((4 * d * E_all + 2 * d * E_cmp) / t_f / 1e12, 1),
                                                  "tensor_frac": round((4 * d * E_all + 2 * d * E_cmp) / t_f / 1e12 / tc_peak, 4)}
            kernel_roofline["backward_kernels"] = {"tflops": round(10 * d * E_all / t_b / 1e12, 1),
                                                   "tensor_frac": round(10 * d * E_all / t_b / 1e12 / tc_peak, 4)}

    # ---- e2e through the public API with host buffers ----
    # Every step copies its inputs (coords, q, k, v, gates, dO) from pinned host memory and reads its
    # results (out, dq, dk, dv, dgates) back to pinned host memory. Copies run on their own streams,
    # double-buffered, so step i's compute overlaps step i+1's H2D and step i-1's D2H (PCIe is full
    # duplex); the clock runs from the first H2D to the last D2H.
    e2e = None
    if not args.no_e2e and not hybrid and not sharded:
        hin = [x.cpu().pin_memory() for x in (c_d, q, k, v, g, do)]
        bi = sum(x.numel() * x.element_size() for x in hin)
        dev_in = [[torch.empty_like(x) for x in (c_d, q, k, v, g, do)] for _ in range(2)]
        dev_out = [[torch.empty_like(out)] + [torch.empty_like(x) for x in grads] for _ in range(2)]
        hout = [[torch.empty_like(x, device="cpu").pin_memory() for x in dev_out[0]] for _ in range(2)]
        bo = sum(x.numel() * x.element_size() for x in hout[0])
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        n_e = args.steps + 2                      # the first two iterations are warm-up
        ev = {key: [torch.cuda.Event() for _ in range(n_e)] for key in ("in", "done", "out")}
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        def read_back(j):   # D2H of step j's results, on the D2H stream after step j is done
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev["done"][j])
                for hx, dx in zip(hout[j % 2], dev_out[j % 2]):
                    hx.copy_(dx, non_blocking=True)
                ev["out"][j].record(s_out)

        # The plan build reads a few counters back to the host (pageable, synchronous); it is issued
        # before the previous step's large D2H so that small read never queues behind it.
        for i in range(n_e):
            slot = i % 2
            if i == 2:
                e0.record(s_in)
            with torch.cuda.stream(s_in):
                if i >= 2:
                    s_in.wait_event(ev["done"][i - 2])            # the step that read this input slot is done
                for hx, dx in zip(hin, dev_in[slot]):
                    dx.copy_(hx, non_blocking=True)
                ev["in"][i].record(s_in)
            st.wait_event(ev["in"][i])
            if i >= 2:
                st.wait_event(ev["out"][i - 2])                   # this output slot has been read back
            cc, qq, kk, vv, gg, dd = dev_in[slot]
            step(qq, kk, vv, gg, dd, dev_out[slot][0], tuple(dev_out[slot][1:]), cc,
                 after_build=(lambda j=i - 1: read_back(j)) if i >= 1 else None)
            ev["done"][i].record(st)
        read_back(n_e - 1)
        e1.record(s_out)
        torch.cuda.synchronize(dev)
        e_ms = e0.elapsed_time(e1) / args.steps
        e_ms = max_over_ranks(e_ms, dev)
        e2e = {"value": round(e_ms / shapes_per_step, 4), "unit": UNIT, "h2d_bytes_per_step": int(bi),
               "d2h_bytes_per_step": int(bo),
               "method": "pinned host buffers; H2D / compute / D2H on three streams, double-buffered; "
                         "timed from the first H2D to the last D2H over the K steps"}

    # ---- full-attention comparator on the same box (context: "speedup vs full attention") ----
    full = None
    if not args.no_full and rank == 0:
        # every shape of the batch timed at its own token count (cost grows with n^2), summed
        for n_b in sorted(set(int(x) for x in ntok_b)):
            r_b = full_attention_time(torch, dev, n_b, H, h_kv, d, tdt)
            mult = int(np.sum(ntok_b == n_b))
            if full is None:
                full = dict(r_b, tokens=[n_b] * mult, flops=r_b["flops"] * mult)
                full["others"] = {kk: vv * mult if kk.endswith("_ms") else vv for kk, vv in r_b["others"].items()}
                if "fwd_bwd_ms" in r_b:
                    full["fwd_bwd_ms"] = r_b["fwd_bwd_ms"] * mult
                continue
            full["tokens"] += [n_b] * mult
            full["flops"] += r_b["flops"] * mult
            if "fwd_bwd_ms" in r_b and "fwd_bwd_ms" in full:
                full["fwd_bwd_ms"] = round(full["fwd_bwd_ms"] + r_b["fwd_bwd_ms"] * mult, 3)
            for kk, vv in r_b["others"].items():
                if kk.endswith("_ms") and kk in full["others"]:
                    full["others"][kk] = round(full["others"][kk] + vv * mult, 3)
        if full is not None and batch > 1:
            full["note"] = "each shape timed at its own token count; times summed over the batch"

    # ---- context: sparse 3D window attention alone (SSA_WINDOW_ONLY; the SS-VAE layer) on the same tokens ----
    win = None
    if rank == 0 and used_tc and not sharded and not args.no_window:
        wcfg = ssa.AttnCfg(h_q=H, h_kv=h_kv, d=d, top_k=T, dtype=tdt, flags=ssa.SSA_WINDOW_ONLY)
        plan_w = ssa.ssa_build_blocks(c_d, grid, batch, *ms)
        wt = []
        for i in range(8):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _, sv = ssa.ssa_forward(plan_w, wcfg, q, k, v, g, out=out)
            ssa.ssa_backward(plan_w, wcfg, sv, q, k, v, g, do, grads=grads)
            e1.record(st)
            if i >= 3:
                wt.append((e0, e1))
        torch.cuda.synchronize(dev)
        win = {"impl": "SSA_WINDOW_ONLY (sparse 3D window attention alone, fwd+bwd, same tokens and windows)",
               "fwd_bwd_ms": round(float(np.mean([a.elapsed_time(b) for a, b in wt])) / batch, 4)}

    # ---- context: the learned delta (R17) + gate projection (R18) variant of the same step, C = 1024
    # input features (the DiT width); random weights (trained ones are out of scope) ----
    learned_ctx = None
    if rank == 0 and used_tc and not sharded and not hybrid and not args.no_learned:
        C = 1024
        gen = torch.Generator(device=dev).manual_seed(5)
        m3 = cfg["m_cmp"] ** 3
        eye = torch.eye(d, device=dev)
        Wk = eye + 0.05 * torch.randn(m3, h_kv, d, d, device=dev, generator=gen)
        Wv = eye + 0.05 * torch.randn(m3, h_kv, d, d, device=dev, generator=gen)
        bk = torch.zeros(h_kv, d, device=dev)
        xf = torch.randn(q.shape[0], C, device=dev, generator=gen).to(tdt)
        Wg = torch.randn(C, 3 * H, device=dev, generator=gen) / math.sqrt(C)
        bg = torch.zeros(3 * H, device=dev)
        lcfg = ssa.AttnCfg(h_q=H, h_kv=h_kv, d=d, top_k=T, dtype=tdt, learned=ssa.Learned(
            conv_k_w=Wk, conv_k_b=bk, conv_v_w=Wv, conv_v_b=bk, x=xf, gate_w=Wg, gate_b=bg))
        lt = []
        ssa.profile_reset()
        ssa.profile_enable(True)
        for i in range(8):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            plan_l = ssa.ssa_build_blocks(c_d, grid, batch, *ms)
            _, sv = ssa.ssa_forward(plan_l, lcfg, q, k, v, None, out=out)
            ssa.ssa_backward(plan_l, lcfg, sv, q, k, v, None, do)
            e1.record(st)
            if i >= 3:
                lt.append((e0, e1))
        torch.cuda.synchronize(dev)
        ssa.profile_enable(False)
        lk = {}
        for kn in ("k_pool_learned", "k_gate_proj"):
            t_, n_ = ssa.profile_read(kn)
            if n_:
                lk[kn] = round(t_ / n_, 4)
        ssa.profile_reset()
        l_ms = float(np.mean([a.elapsed_time(b) for a, b in lt]))
        learned_ctx = {"impl": "learned delta (sparse conv kernel = stride = m_cmp + mean pool, R17) and gate "
                               "projection from C = 1024 features (R18), fwd+bwd incl. weight gradients",
                       "fwd_bwd_ms": round(l_ms / batch, 4), "extra_ms_vs_plain": round((l_ms - ms_per_step) / batch, 4),
                       "kernel_ms": lk}

    # ---- context: the paper's DiT attention layout (2 kv groups x 16 heads, head dim 32) on the
    # same tokens (tcgen05 kernels, heads zero-padded to 64 inside the library) ----
    paper_ctx = None
    if rank == 0 and used_tc and not sharded and not hybrid and not args.no_learned:
        gen = torch.Generator(device=dev).manual_seed(6)
        Hp, dp = 32, 32
        tp = [torch.randn(q.shape[0], hh, dp, device=dev, generator=gen).to(tdt) for hh in (Hp, h_kv, h_kv)]
        gp = torch.sigmoid(torch.randn(q.shape[0], Hp, 3, device=dev, generator=gen)).to(tdt)
        dop = torch.randn(q.shape[0], Hp, dp, device=dev, generator=gen).to(tdt)
        pcfg = ssa.AttnCfg(h_q=Hp, h_kv=h_kv, d=dp, top_k=T, dtype=tdt)
        pt = []
        for i in range(6):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            plan_p = ssa.ssa_build_blocks(c_d, grid, batch, *ms)
            _, sv = ssa.ssa_forward(plan_p, pcfg, *tp, gp)
            ssa.ssa_backward(plan_p, pcfg, sv, *tp, gp, dop)
            e1.record(st)
            if i >= 2:
                pt.append((e0, e1))
        torch.cuda.synchronize(dev)
        paper_ctx = {"impl": "paper DiT layout H = 32 (h_kv = 2), d = 32 (P:272), same tokens, tcgen05 (d padded to 64)",
                     "fwd_bwd_ms": round(float(np.mean([a.elapsed_time(b) for a, b in pt])) / batch, 4),
                     "path": "tcgen05" if sv.used_tcgen05 else "simt"}

    # ---- context: the paper's exact per-token selection (Alg. 1, I in R^{N x h_kv x T}, P:182 / P:188): the
    # same tokens with query blocks of one token (m_q = 1) on the tcgen05 kernels ----
    tok_ctx = None
    if rank == 0 and used_tc and not sharded and not hybrid and not args.no_learned:
        ms1 = tuple(ms[:3]) + (1,)
        tt = []
        for i in range(6):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            plan_t = ssa.ssa_build_blocks(c_d, grid, batch, *ms1)
            _, sv = ssa.ssa_forward(plan_t, acfg, q, k, v, g, out=out)
            ssa.ssa_backward(plan_t, acfg, sv, q, k, v, g, do)
            e1.record(st)
            if i >= 2:
                tt.append((e0, e1))
        torch.cuda.synchronize(dev)
        t_ms = float(np.mean([a.elapsed_time(b) for a, b in tt])) / batch
        tok_ctx = {"impl": "per-token selection m_q = 1 (Alg. 1 granularity), same tokens and heads, tcgen05 "
                           "(selection forward and dQ as per-block passes merged by LSE, window / compressed keys "
                           "on sub-groups of tokens, packed KV-outer row tiles)",
                   "fwd_bwd_ms": round(t_ms, 4), "ratio_vs_query_block_path": round(t_ms / ms_per_step, 2),
                   "path": "tcgen05" if sv.used_tcgen05 else "simt"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args, cfg, coords, grid, batch, inp, value)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": False,
            "scaling": "strong" if (sharded or hybrid) else "weak", "vs_baseline": None,
            "dtype": "bf16" if tdt == torch.bfloat16 else "f32",
            "data": "synthetic (sphere-shell occupancy, N(0,1) q/k/v/dO, sigmoid(N(0,1)) gates; ssa_workload)",
            "config": {"workload": f"{args.config}: 128^3 latent (1024^3 res) sphere shell, {N} tokens x {batch} shape(s)/rank, "
                                   f"H={H} (h_kv={h_kv}), d={d}, m_cmp/m_slc/m_win/m_q={ms}, T={T}",
                       "tokens_per_shape": int(np.max(ntok_b)), "shapes_per_rank": batch,
                       "parallelism": (f"query-block shards x{world} ({args.backend}: pooled-key all-reduce, K/V "
                                       "all-gather overlapped with the compression branch, dK/dV reduce-scatter)"
                                       if sharded else
                                       (f"hybrid x{world}: batch cost line cut into {world} pieces; whole shapes "
                                        "per rank, cut shapes query-block sharded over sub-groups" if hybrid else
                                        f"shape-parallel x{world} (no data-path collective)")),
                       "l2": "flushed between timed steps (256 MB write)", "path": "tcgen05" if used_tc else "simt"},
            "clocks": clocks, "gpu_launches": int(launches), "roofline": roofline, "kernel_ms": kernel_ms,
            "kernel_roofline": kernel_roofline,
            "work": {"E_cmp": E_cmp, "E_slc": E_slc, "E_win": E_win},
            "e2e": e2e, "cpu_baseline": cpu,
        }
        if win:
            line["window_attention"] = win
        if learned_ctx:
            line["learned_delta_gates"] = learned_ctx
        if paper_ctx:
            line["paper_layout_d32"] = paper_ctx
        if tok_ctx:
            line["per_token_m_q1"] = tok_ctx
        if hybrid_info:
            line["config"]["hybrid_plan"] = hybrid_info["plan"]
        if full:
            line["full_attention"] = full
            if "fwd_bwd_ms" in full:
                line["speedup_vs_full_attention"] = round(full["fwd_bwd_ms"] / ms_per_step, 2)
            for key, val in full.get("others", {}).items():
                if key.endswith("_ms"):
                    line.setdefault("speedup_vs", {})[key[:-3]] = round(val / ms_per_step, 2)
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def full_attention_time(torch, dev, n, H, h_kv, d, dt):
    """Dense non-causal attention over all n tokens, fwd+bwd, GQA (context only, SURVEY 8d comparators):
    torch SDPA default dispatch, SDPA pinned to the cuDNN backend, flash_attn (FA2) and the FA4 CuTe-DSL
    sm100 kernels (vllm.vllm_flash_attn.cute) when they run here."""
    import torch.nn.functional as F
    q = torch.randn(1, H, n, d, device=dev, dtype=dt, requires_grad=True)
    k = torch.randn(1, h_kv, n, d, device=dev, dtype=dt, requires_grad=True)
    v = torch.randn(1, h_kv, n, d, device=dev, dtype=dt, requires_grad=True)
    go = torch.randn(1, H, n, d, device=dev, dtype=dt)

    def timed(run, reps=3):
        for _ in range(2):
            run()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize(dev)
        return round(e0.elapsed_time(e1) / reps, 3)

    res = {"impl": "torch SDPA (GQA, non-causal, bf16)", "tokens": n, "flops": 4.0 * n * n * H * d * 3.5}
    try:
        res["fwd_bwd_ms"] = timed(lambda: F.scaled_dot_product_attention(q, k, v, enable_gqa=True).backward(go))
    except Exception as ex:  # comparator is context only
        res["error"] = str(ex)[:200]
    others = {}
    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel

        def cudnn():
            with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                kk = k.repeat_interleave(H // h_kv, dim=1)
                vv = v.repeat_interleave(H // h_kv, dim=1)
                F.scaled_dot_product_attention(q, kk, vv).backward(go)
        others["cudnn_sdpa_ms"] = timed(cudnn)
    except Exception as ex:
        others["cudnn_sdpa_error"] = str(ex)[:160]
    try:
        from flash_attn import flash_attn_func
        qf = q.detach().transpose(1, 2).contiguous().requires_grad_(True)
        kf = k.detach().transpose(1, 2).contiguous().requires_grad_(True)
        vf = v.detach().transpose(1, 2).contiguous().requires_grad_(True)
        gof = go.transpose(1, 2).contiguous()
        others["flash_attn2_ms"] = timed(lambda: flash_attn_func(qf, kf, vf).backward(gof))
    except Exception as ex:
        others["flash_attn2_error"] = str(ex)[:160]
    try:
        # FA4 (CuTe DSL, sm100: tcgen05 / TMEM), vendored by vllm — the strongest full-attention kernel here
        from vllm.vllm_flash_attn.cute.interface import flash_attn_func as fa4
        q4 = q.detach().transpose(1, 2).contiguous().requires_grad_(True)
        k4 = k.detach().transpose(1, 2).contiguous().requires_grad_(True)
        v4 = v.detach().transpose(1, 2).contiguous().requires_grad_(True)
        go4 = go.transpose(1, 2).contiguous()

        def fa4_step():
            o4 = fa4(q4, k4, v4, causal=False)
            (o4[0] if isinstance(o4, tuple) else o4).backward(go4)
        others["flash_attn4_cute_ms"] = timed(fa4_step)
    except Exception as ex:
        others["flash_attn4_cute_error"] = str(ex)[:160]
    res["others"] = others
    return res


_OS = {}   # oracle state shared with forked sample workers (copy-on-write)


def _oracle_one_q(Q):
    """The oracle's per-query-block work, as oracle.ssa_forward / ssa_backward do it for one Q: compression
    attention, Eq. 8 scores, top-k, selection + window attention, gated sum, and the three branch
    backwards, for every kv group."""
    import oracle as O
    st = _OS
    plan, cfg = st["plan"], st["cfg"]
    qs, ks, vs, gs, dos, k_cmp, v_cmp = (st[x] for x in ("qs", "ks", "vs", "gs", "dos", "k_cmp", "v_cmp"))
    H, h_kv, d = cfg["H"], cfg["h_kv"], cfg["d"]
    h_s = H // h_kv
    scale = 1.0 / math.sqrt(d)
    Cq, Cs, Cw = plan.offsets["q"], plan.offsets["slc"], plan.offsets["win"]
    a, b_ = int(Cq[Q]), int(Cq[Q + 1])
    bi = int(plan.sorted_coords[a, 0])
    c0, c1 = int(plan.batch_blocks["cmp"][bi]), int(plan.batch_blocks["cmp"][bi + 1])
    s0 = int(plan.batch_blocks["slc"][bi])
    w = int(plan.tok_block["win"][a])
    for g in range(h_kv):
        rows = qs[a:b_, g * h_s:(g + 1) * h_s].reshape(-1, d)
        drow = dos[a:b_, g * h_s:(g + 1) * h_s].reshape(-1, d)
        wt = gs[a:b_, g * h_s:(g + 1) * h_s].reshape(-1, 3)
        oc, _, pc = O.dense_attention(rows, k_cmp[c0:c1, g], v_cmp[c0:c1, g], scale)
        per = pc.sum(axis=0)
        sc = np.zeros(int(plan.batch_blocks["slc"][bi + 1]) - s0)
        np.add.at(sc, plan.cmp_to_slc[c0:c1] - s0, per)
        sel = O.topk_select(sc, cfg["T"], base=s0)
        kt = np.concatenate([np.arange(Cs[x], Cs[x + 1]) for x in sel if x >= 0])
        os_, _, ps = O.dense_attention(rows, ks[kt, g], vs[kt, g], scale)
        wa, wb = int(Cw[w]), int(Cw[w + 1])
        ow, _, pw = O.dense_attention(rows, ks[wa:wb, g], vs[wa:wb, g], scale)
        _ = wt[:, 0:1] * oc + wt[:, 1:2] * os_ + wt[:, 2:3] * ow
        O.dense_attention_backward(rows, k_cmp[c0:c1, g], v_cmp[c0:c1, g], pc, oc, wt[:, 0:1] * drow, scale)
        O.dense_attention_backward(rows, ks[kt, g], vs[kt, g], ps, os_, wt[:, 1:2] * drow, scale)
        O.dense_attention_backward(rows, ks[wa:wb, g], vs[wa:wb, g], pw, ow, wt[:, 2:3] * drow, scale)


def _oracle_worker(Qs):
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):           # one worker process per core, BLAS single-threaded
        t = time.perf_counter()
        for Q in Qs:
            _oracle_one_q(int(Q))
        return time.perf_counter() - t


def host_cores():
    return len(os.sched_getaffinity(0))


def oracle_sample(cfg, coords, grid, batch, inp, n_sample: int, seed: int = 0):
    """Time the float64 oracle (as it stands) on a bounded sample of the workload, one worker process per
    host core: the full block build and pooling (sequential, once), then the per-query-
    block work for n_sample random query blocks dealt evenly to the workers. Returns (build s, parallel
    wall s of the sample, sampled blocks, total blocks, workers); the step estimate is
    build + wall * total / sampled."""
    import multiprocessing as mp
    import oracle as O
    t0 = time.perf_counter()
    kw = dict(m_cmp=cfg["m_cmp"], m_slc=cfg["m_slc"], m_win=cfg["m_win"], m_q=cfg["m_q"])
    plan = O.block_build(coords, grid, batch, **kw)
    P = plan.perm
    qs, ks, vs = inp.q[P].astype(np.float64), inp.k[P].astype(np.float64), inp.v[P].astype(np.float64)
    gs, dos = inp.gates[P].astype(np.float64), inp.dout[P].astype(np.float64)
    k_cmp, v_cmp = O.compress(plan, ks), O.compress(plan, vs)
    t_build = time.perf_counter() - t0
    _OS.update(plan=plan, cfg=cfg, qs=qs, ks=ks, vs=vs, gs=gs, dos=dos, k_cmp=k_cmp, v_cmp=v_cmp)
    nq = plan.n_blocks("q")
    rng = np.random.Generator(np.random.PCG64(seed))
    sample = rng.choice(nq, size=min(n_sample, nq), replace=False)
    workers = max(1, min(host_cores(), len(sample)))
    parts = [x for x in np.array_split(sample, workers) if len(x)]
    t1 = time.perf_counter()
    with mp.get_context("fork").Pool(len(parts)) as pool:
        pool.map(_oracle_worker, parts)
    t_q = time.perf_counter() - t1
    _OS.clear()
    return t_build, t_q, len(sample), nq, workers


def cpu_baseline(args, cfg, coords, grid, batch, inp, gpu_value):
    n_sample = args.cpu_sample or 4 * host_cores()
    t_build, t_q, ns, nq, workers = oracle_sample(cfg, coords, grid, batch, inp, n_sample)
    est_s = t_build + t_q * nq / ns
    res = {"value": round(est_s * 1e3 / batch, 1), "unit": UNIT, "cores": workers, "kind": "oracle",
           "sample": f"float64 numpy oracle, {workers} worker processes (one per host core, BLAS 1 thread each): full "
                     f"block build + pool ({t_build:.1f} s) and fwd+bwd of {ns} random query blocks of {nq} "
                     f"({t_q:.1f} s wall), extrapolated to all query blocks"}
    if args.cpu_check_c2 and args.config != "C2":
        # the extrapolation, checked where the oracle finishes: C2 sampled the same way vs every query block
        from ssa_workload import CONFIGS, config_coords, make_inputs
        c2 = CONFIGS["C2"]
        cc, gg, bb = config_coords("C2")
        inp2 = make_inputs(cc, gg, bb, c2["H"], c2["h_kv"], c2["d"], c2["dtype"], seed=c2["seed"])
        tb, tq, ns2, nq2, w2 = oracle_sample(c2, cc, gg, bb, inp2, n_sample)
        tb_f, tq_f, _, nq_f, _ = oracle_sample(c2, cc, gg, bb, inp2, 10 ** 9)     # every query block
        res["c2_check"] = {"sampled_estimate_s": round(tb + tq * nq2 / ns2, 2), "all_blocks_s": round(tb_f + tq_f, 2),
                           "note": f"C2 (24 808 tokens): the same {w2}-process oracle on {ns2} sampled query blocks "
                                   f"(extrapolated) vs on all {nq_f} query blocks (no extrapolation)"}
    return res


def reference_arm(args, rank, world):
    """--impl reference: the oracle as it stands, on the host cores, bounded sample per step."""
    if rank != 0:
        return
    from ssa_workload import make_inputs
    cfg, coords, grid, batch = workload(args.config, 0, 1)
    inp = make_inputs(coords, grid, batch, cfg["H"], cfg["h_kv"], cfg["d"], cfg["dtype"], seed=cfg["seed"])
    per_step = []
    workers = 1
    n_sample = args.cpu_sample or 2 * host_cores()
    for i in range(args.warmup + args.steps):
        t_build, t_q, ns, nq, workers = oracle_sample(cfg, coords, grid, batch, inp, n_sample, seed=i)
        if i >= args.warmup:
            per_step.append(t_build + t_q * nq / ns)
    v = float(np.mean(per_step)) * 1e3 / batch
    line = {"metric": METRIC, "value": round(v, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(v * batch, 1), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (ssa_workload)", "impl": "reference",
            "config": {"workload": f"{args.config} (oracle sample, extrapolated)", "parallelism": f"{workers} host processes"},
            "cpu_baseline": {"value": round(v, 1), "unit": UNIT, "cores": workers, "kind": "oracle",
                             "sample": f"per step: full block build/pool + {n_sample} random query blocks on {workers} "
                                       "worker processes (one per core), extrapolated to all query blocks"},
            "e2e": {"value": round(v, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
