#!/bin/bash
# A/B of an environment switch in one GPU session (alternating runs): profiles/ab_env.sh "<ENV=val>" <rounds> <bench args...>
E=$1; R=$2; shift 2
for r in $(seq 1 $R); do
  for mode in base alt; do
    if [ $mode = alt ]; then env $E python bench.py --no-cpu-baseline --no-extras --no-configs "$@" 2>/dev/null | tail -n 1 > /tmp/ab_line.json
    else python bench.py --no-cpu-baseline --no-extras --no-configs "$@" 2>/dev/null | tail -n 1 > /tmp/ab_line.json; fi
    python - "$mode" <<'PY'
import json,sys
l=json.loads(open('/tmp/ab_line.json').read())
b=l.get('build') or {}
print(sys.argv[1], l['config'].get('workload','')[:3], 'q/s', round(l['value']/1e6,1), 'insert_l_ms', round(b.get('insert_l_ms',0),3),
      'buildveb_ms', round(b.get('buildveb_ms',0),3), 'ins', round((l.get('insert_l_points_per_s') or 0)/1e6,1), 'era', round((l.get('erase_l_points_per_s') or 0)/1e6,1))
PY
  done
done
