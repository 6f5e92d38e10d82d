"""Summarise an ncu source page (SASS) export: instruction share and stall
share per straight-line region.  Usage:
  ncu -i X.ncu-rep --page source --csv --print-source sass > /tmp/s.csv
  python profiles/sass_hot.py /tmp/s.csv [min_pct]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
minp = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
ai, si = h.index("Address"), h.index("Source")
st, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
ti = sum(float(r[ie] or 0) for r in data)
ts = sum(float(r[st] or 0) for r in data)
regions, cur = [], None
for r in data:
    i = float(r[ie] or 0)
    if cur is None or abs(i - cur["last"]) > 1e-9 * ti + 0.5:
        cur = {"start": r[ai][-5:], "n": 0, "ins": 0.0, "stall": 0.0, "last": i, "first": r[si][:60]}
        regions.append(cur)
    cur["n"] += 1
    cur["ins"] += i
    cur["stall"] += float(r[st] or 0)
print(f"total instructions {ti:.4g}, stall samples {ts:.4g}")
for g in regions:
    if 100 * g["ins"] / ti >= minp or 100 * g["stall"] / ts >= minp:
        print(f"{g['start']:>6s} n={g['n']:4d} exec/instr={g['last']:.3g} instr%={100*g['ins']/ti:5.1f} stall%={100*g['stall']/ts:5.1f}  {g['first']}")
