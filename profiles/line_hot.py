"""Per-CUDA-source-line instruction and stall shares from an ncu capture.
  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > /tmp/cs.csv
  python profiles/line_hot.py /tmp/cs.csv [min_pct]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
minp = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
fname, hdr, agg = "?", None, {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    ie = hdr.index("Instructions Executed")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        key = (fname, int(r[0]))
    except ValueError:
        continue
    a = agg.setdefault(key, [0.0, 0.0, r[1].strip()[:90]])
    a[0] += float(r[ie] or 0) if r[ie] not in ("-", "") else 0
    a[1] += float(r[st] or 0) if r[st] not in ("-", "") else 0
ti = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values())
print(f"total warp instructions {ti:.4g}, stall samples {ts:.4g}")
for (f, l), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    if 100 * i / ti >= minp or 100 * s / ts >= minp:
        print(f"{f}:{l:<5d} instr {100*i/ti:5.1f}%  stall {100*s/ts:5.1f}%  {src}")
