#!/bin/bash
# like capture_all.sh for a subset: profiles/capture_some.sh <tag> "<name> <what> <regex> [replay-mode]" ...
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
for spec in "$@"; do
  set -- $spec
  name=$1; what=$2; rx=$3; mode=${4:-kernel}
  rx=${rx//_SP_/ }
  timeout 900 ncu -f --set full --import-source on --clock-control none --replay-mode $mode --kernel-name-base demangled \
    -k "regex:$rx" -c 1 -o /tmp/ncu_$name python profiles/ncu_drive.py $what > $OUT/$name.log 2>&1 || echo "capture $name failed"
  tail -4 $OUT/$name.log
  [ -f /tmp/ncu_$name.ncu-rep ] && python profiles/ncu_digest.py /tmp/ncu_$name.ncu-rep > $OUT/$name.json 2>&1
  [ -f /tmp/ncu_$name.ncu-rep ] && [ $(stat -c %s /tmp/ncu_$name.ncu-rep) -lt 8000000 ] && cp /tmp/ncu_$name.ncu-rep $OUT/
done
echo capture_some done
