#!/bin/bash
# K1 A/B of several libgkbdl.so builds (alternating runs, one GPU session) with the
# instrumented pass's counters: value, K1 ms, warp-level insert events, lane accepts.
#   profiles/abk.sh "<libA.so> <libB.so> ..." <rounds> <bench args...>
LIBS=$1; R=$2; shift 2
for r in $(seq 1 $R); do
  for L in $LIBS; do
    GK_LIB=$L python bench.py --no-cpu-baseline --no-extras --no-configs "$@" 2>/dev/null | tail -n 1 | python -c "
import json,sys
l=json.loads(sys.stdin.read())
r=l.get('roofline') or {}
c=r.get('counters') or {}
print('$L'.split('/')[-2], 'cfg', l['config'].get('workload','')[:3], round(l['value']/1e6,1), 'Mq/s k1_ms', round(r.get('k1_ms',0),3),
      'wev', c.get('warp_inserts'), 'ins', c.get('inserts'), 'wl', c.get('warp_leaves'), 'wlp', c.get('warp_leaf_points'))"
  done
done
