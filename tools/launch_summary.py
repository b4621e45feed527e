"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel total ms, share, launches.
python tools/launch_summary.py launches.csv [title]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
unit_i = h.index("Metric Unit") if "Metric Unit" in h else None
agg = collections.defaultdict(lambda: [0.0, 0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    unit = r[unit_i] if unit_i is not None else "ns"
    v = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
    name = r[ki].split("(")[0]
    agg[name][0] += v
    agg[name][1] += 1
tot = sum(a[0] for a in agg.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print(f"total device time {tot:.2f} ms over {sum(a[1] for a in agg.values())} launches\n")
print(f"{'ms':>9} {'share':>6} {'launches':>8}  kernel")
for k, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{v:9.3f} {100 * v / tot:5.1f}% {c:8d}  {k}")
