"""Summarise an ncu --set full report (raw page) and a launch-list CSV into markdown + json."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(rep, launches, tag):
    hdr, units, rows = raw_rows(rep)
    ix = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}

    def mb(r, k):
        try:
            return float(r[ix[k]]) * scale.get(units[ix[k]], 1.0)
        except (KeyError, ValueError):
            return 0.0

    def g(r, k, default=""):
        return r[ix[k]] if k in ix else default

    lines = [f"# ncu summary {tag}", "", f"source: `{rep}` (ncu --set full --clock-control none --import-source on),"
             f" launch list `{launches}`", "",
             "| kernel | time ms | tensor pipe % | MUFU(xu) % | DRAM read MB | DRAM write MB | L2 % | regs | top stalls |",
             "|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for r in rows:
        name = g(r, "Kernel Name").split("(")[0].replace("ssa::<unnamed>::", "")
        if "mode" in name:
            pass
        st = []
        for h, i in ix.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        st.sort(reverse=True)
        tot = sum(v for v, _ in st) or 1
        grid = g(r, "Grid Size") if "Grid Size" in ix else ""
        rd = mb(r, "dram__bytes_read.sum")
        wr = mb(r, "dram__bytes_write.sum")
        unit_r = hdr  # units row not kept; ncu reports dram bytes in the unit of row 1
        lines.append(f"| {name} | {float(g(r, 'gpu__time_duration.sum', '0')):.3f} | "
                     f"{g(r, 'TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed')[:5]} | "
                     f"{g(r, 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active')[:5]} | {rd:.1f} | {wr:.1f} | "
                     f"{g(r, 'lts__throughput.avg.pct_of_peak_sustained_elapsed')[:5]} | {g(r, 'launch__registers_per_thread')} | "
                     + ", ".join(f"{n} {100*v/tot:.0f}%" for v, n in st[:4]) + " |")
        key = name if name not in traffic else f"{name}#{sum(1 for k in traffic if k.split('#')[0] == name)}"
        traffic[key] = (rd + wr) * 1e6   # bytes per launch (repeated kernel names: #1, #2 ... in launch order)
    # launch list: device time share per kernel over the captured steps
    agg, cnt = defaultdict(float), defaultdict(int)
    text = open(launches).read().splitlines()
    start = [i for i, l in enumerate(text) if l.startswith('"ID"')][0]
    lr = list(csv.reader(text[start:]))
    h = lr[0]
    for r in lr[1:]:
        try:
            v = float(r[h.index("Metric Value")].replace(",", ""))
        except (ValueError, IndexError):
            continue
        n = r[h.index("Kernel Name")].split("(")[0].replace("ssa::<unnamed>::", "").replace("void ", "")
        agg[n] += v / 1e6
        cnt[n] += 1
    total = sum(agg.values())
    lines += ["", "## launch list (ncu gpu__time_duration, cold-cache serialised; compare shares)", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for n, v in sorted(agg.items(), key=lambda x: -x[1]):
        lines.append(f"| {n} | {cnt[n]} | {v:.3f} | {100*v/total:.1f}% |")
    lines.append(f"| **all** | {sum(cnt.values())} | {total:.3f} | 100% |")
    print("\n".join(lines))
    return traffic


if __name__ == "__main__":
    t = main(sys.argv[1], sys.argv[2], sys.argv[3])
    if len(sys.argv) > 4:
        json.dump({k: v for k, v in t.items()}, open(sys.argv[4], "w"), indent=1)
