#!/bin/bash
# A/B/... timing of several builds of libgkbdl.so in one GPU session (alternating runs).
#   profiles/abn.sh "<libA.so> <libB.so> ..." <rounds> <bench args...>
LIBS=$1; R=$2; shift 2
for r in $(seq 1 $R); do
  for L in $LIBS; do
    GK_LIB=$L python bench.py --no-cpu-baseline --no-configs "$@" 2>/dev/null | tail -n 1 | python -c "
import json,sys
l=json.loads(sys.stdin.read())
b=l.get('build') or {}
e=(l.get('e2e') or {}).get('value',0)
print('$L'.split('/')[-2], round(l['value']/1e6,1), 'Mq/s', 'insert_l_ms', round(b.get('insert_l_ms',0),2), 'buildveb_ms', round(b.get('buildveb_ms',0),2), 'e2e', round(e/1e6,1), 'ins', round((l.get('insert_l_points_per_s') or 0)/1e6,1), 'era', round((l.get('erase_l_points_per_s') or 0)/1e6,1))"
  done
done
