"""Summarise ncu outputs into profiles/<name>.md: launch-list shares per kernel and the key
counters of a --set full capture.  Usage: python tools/ncu_summary.py <launches.csv> <rep.ncu-rep> <out.md> [title]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total µs | share |", "|---|---|---|---|"]
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f}% |")
    return "\n".join(out), tot


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    cols = [m for m in METRICS if m in hdr]
    out = ["| kernel | grid | " + " | ".join(c.split(".")[0] + f" ({units[hdr.index(c)]})" for c in cols if c != "launch__grid_size") + " |",
           "|---|---|" + "---|" * (len(cols) - (1 if "launch__grid_size" in cols else 0))]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        grid = r[hdr.index("Grid Size")] if "Grid Size" in hdr else ""
        out.append(f"| `{name}` | {grid} | " + " | ".join(r[hdr.index(c)] for c in cols if c != "launch__grid_size") + " |")
    return "\n".join(out)


if __name__ == "__main__":
    lc, rep, dst = sys.argv[1:4]
    title = sys.argv[4] if len(sys.argv) > 4 else dst
    t, tot = launches(lc)
    body = f"# {title}\n\n## Launch list (ncu gpu__time_duration, cold-cache, serialised; compare shares)\n\nTotal {tot:.1f} µs\n\n{t}\n\n## Full capture (--set full) of the top kernel\n\n{full(rep)}\n"
    open(dst, "w").write(body)
    print(body)
