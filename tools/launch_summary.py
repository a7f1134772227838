"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel launches, total
and mean device time, and share of the listed time.  usage: launch_summary.py CSV [steps]"""
import csv, sys
from collections import defaultdict
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    try:
        v = float(r[i_val].replace(",", ""))
    except (ValueError, IndexError):
        continue
    n = r[i_name].split("(")[0].replace("void ", "")
    agg[n][0] += 1
    agg[n][1] += v
tot = sum(v for _, v in agg.values())
print(f"{'kernel':55s} {'launches':>8s} {'total us':>10s} {'share':>6s} {'us/launch':>10s}")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:55]:55s} {c:8d} {v / 1e3:10.1f} {100 * v / tot:5.1f}% {v / c / 1e3:10.2f}")
print(f"listed device time {tot / 1e3:.1f} us = {tot / 1e3 / steps:.1f} us per step over {steps} steps")
