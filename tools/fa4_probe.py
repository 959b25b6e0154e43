"""Probe the FA4 (CuTe DSL sm100) full-attention comparator at a small and at the C3 size."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda")
for n in (8192, 122552):
    t = time.time()
    r = bench.full_attention_time(torch, dev, n, 16, 2, 64, torch.bfloat16)
    print(n, round(time.time() - t, 1), "s", r.get("fwd_bwd_ms"), r["others"], flush=True)
