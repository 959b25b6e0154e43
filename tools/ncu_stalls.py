"""Per-region warp-stall breakdown from `ncu -i REP --page source --csv --print-source sass`.

Usage: python tools/ncu_stalls.py SRC.csv [top_n]
Prints the total stall-reason mix and the top-N sampled SASS instructions with their dominant reasons."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
lines = []
for i, r in enumerate(data):
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    rc = {k: int(r[ix[k]] or 0) for k in reasons}
    tot.update(rc)
    lines.append((s, i, r[ix["Source"]].strip(), rc))
allS = sum(tot.values())
print("total samples", allS)
for k, v in tot.most_common(10):
    print(f"  {k:28s} {v / allS:6.1%}")
print()
for s, i, src, rc in sorted(lines, reverse=True)[:top_n]:
    best = ", ".join(f"{k[6:]}={v}" for k, v in Counter(rc).most_common(3) if v)
    print(f"{i:5d} {s:7d} {src[:60]:60s} {best}")
