#!/bin/bash
# per-launch device times (ncu, serialised) of the kernels matching a regex while running a driver
#   profiles/launch_times.sh <regex> <out.csv> <command...>
RX=$1; OUT=$2; shift 2
ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none \
  --kernel-name-base demangled -k "regex:$RX" --csv "$@" 2>/dev/null | grep '^"' > $OUT
python - $OUT <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
ki, mi, vi, ii, si = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Stream"))
cur = {}
for r in rows[1:]:
    if len(r) < len(h):
        continue
    cur.setdefault(int(r[ii]), {"k": r[ki].split("(")[0].replace("void unnamed>::", ""), "s": r[si]})[r[mi]] = r[vi]
for i, d in sorted(cur.items()):
    print(i, d["s"], d["k"], round(float(d.get("gpu__time_duration.sum", 0)) / 1e3, 1), "us  issue%",
          d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"), "insts", d.get("smsp__inst_executed.sum"))
PY
