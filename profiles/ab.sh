#!/bin/bash
# A/B timing of two builds of libgkbdl.so in one GPU session (alternating runs).
#   profiles/ab.sh <libA.so> <libB.so> <bench args...>
# prints value / build numbers per run; run on a GPU box.
A=$1; B=$2; shift 2
for r in 1 2; do
  for L in "$A" "$B"; do
    GK_LIB=$L python bench.py --no-cpu-baseline --no-configs "$@" 2>/dev/null | tail -n 1 | python -c "
import json,sys
l=json.loads(sys.stdin.read())
b=l.get('build') or {}
print('$L'.split('/')[-2], round(l['value']/1e6,1), 'Mq/s', 'insert_l_ms', round(b.get('insert_l_ms',0),2), 'buildveb_ms', round(b.get('buildveb_ms',0),2), l.get('ops_seconds',''))"
  done
done
