"""Per-kernel DRAM throughput from an ncu metrics CSV (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum; one row per launch): average per launch, achieved GB/s and fraction of the measured
HBM peak (MEASURED_PEAKS.json hbm_gbs). Usage: python tools/ncu_hbm.py launches.csv tag > profiles/hbm_<tag>.md"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = 6650.0
try:
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    src = "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"
except Exception:
    src = "fallback 6650 GB/s"
text = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(text) if l.startswith('"ID"')][0]
rows = list(csv.reader(text[start:]))
h = rows[0]
ik, im, iv, iu = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
         "msecond": 1e-3, "ms": 1e-3}
per = defaultdict(lambda: defaultdict(float))
launches = defaultdict(set)
for r in rows[1:]:
    try:
        v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    except (ValueError, IndexError):
        continue
    name = r[ik].split("(")[0].replace("void ", "").replace("ssa::<unnamed>::", "")
    per[name][r[im]] += v
    launches[name].add(r[0])
print(f"# DRAM throughput per kernel ({sys.argv[2]})\n")
print(f"source: `{os.path.basename(sys.argv[1])}` (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
      f"dram__bytes_write.sum; cold-cache, serialised launches); peak {peak:.0f} GB/s = {src}\n")
print("| kernel | launches | avg us | avg MB (r+w) | GB/s | % of HBM peak |")
print("|---|---|---|---|---|---|")
out = []
for name, m in per.items():
    n = len(launches[name])
    t = m["gpu__time_duration.sum"] / n
    b = (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / n
    out.append((t * n, name, n, t, b))
for _, name, n, t, b in sorted(out, reverse=True):
    gbs = b / t / 1e9 if t > 0 else 0.0
    print(f"| {name} | {n} | {t * 1e6:.1f} | {b / 1e6:.1f} | {gbs:.0f} | {100 * gbs / peak:.1f}% |")
