"""Summarise an ncu source-page CSV (SASS): top instructions by warp-stall samples."""
import csv
import sys


def num(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0


path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[0] != "Address"]
key = "Warp Stall Sampling (All Samples)"
tot = sum(num(d[key]) for d in data)
print(f"total samples {tot:.0f}")
order = sorted(range(len(data)), key=lambda i: -num(data[i][key]))
for i in order[:top]:
    d = data[i]
    s = num(d[key])
    print(f"{s:7.0f} {100*s/max(tot,1):5.1f}%  [{i:5d}] {d['Address']:>6}  {d['Source'][:90]}")
