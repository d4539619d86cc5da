"""Heaviest SASS windows of a kernel by warp-stall samples, from an ncu source
page CSV (ncu -i rep --page source --csv --print-source sass > src.csv).

    python tools/ncu_hot.py src.csv [window] [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
win = int(sys.argv[2]) if len(sys.argv) > 2 else 24
top = int(sys.argv[3]) if len(sys.argv) > 3 else 6
h = rows[1]
data = rows[2:]
isrc, iex, ist = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")


def num(x):
    return int(x) if x.isdigit() else 0


tot = sum(num(r[iex]) for r in data)
tots = sum(num(r[ist]) for r in data)
print(f"total warp instructions {tot}, stall samples {tots}")
w = sorted(((sum(num(r[ist]) for r in data[i:i + win]), sum(num(r[iex]) for r in data[i:i + win]), i)
            for i in range(0, len(data), win)), reverse=True)
for s, e, i in w[:top]:
    print(f"--- rows {i}-{i + win}: samples {s} ({100 * s / tots:.1f}%), instr {e} ({100 * e / tot:.1f}%)")
    for r in data[i:i + win]:
        print(f"{r[ist]:>6} {r[iex]:>9}  {r[isrc].strip()[:80]}")
