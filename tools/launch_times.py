"""Summarize an ncu launch list CSV (--metrics gpu__time_duration.sum --csv):
per-kernel launch count and mean duration.

    python tools/launch_times.py gpurun_out/launches.csv
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = collections.OrderedDict()
for r in rows[start + 1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except (ValueError, IndexError):
        continue
    d.setdefault(r[ki][:70], []).append(v)
tot = sum(sum(v) for v in d.values())
for k, v in d.items():
    print(f"{k:70s} n={len(v):4d} mean_us={sum(v) / len(v) / 1e3:9.2f} share={sum(v) / tot * 100:5.1f}%")
