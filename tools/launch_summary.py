"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list. usage: launch_summary.py csv [steps]"""
import csv, sys
from collections import defaultdict
lines = open(sys.argv[1]).read().splitlines()
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
h = rows[0]
agg, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    try:
        agg[r[h.index("Kernel Name")].split("(")[0].replace("void ", "")] += float(r[h.index("Metric Value")].replace(",", "")) / 1e6
        cnt[r[h.index("Kernel Name")].split("(")[0].replace("void ", "")] += 1
    except (ValueError, IndexError):
        pass
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v / steps:9.3f} ms/step  {cnt[k] / steps:5.1f} launches  {100 * v / tot:5.1f}%  {k}")
print(f"{tot / steps:9.3f} ms/step total")
