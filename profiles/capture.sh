#!/bin/bash
# Round profile capture on a GPU box (run from the repo root, via gpurun):
#   1. the bench command alone (must exit 0 without ncu),
#   2. the launch list of the same command (cold-cache, serialised per-launch times),
#   3. one `ncu --set full` capture of a timed K1 launch (k_knn, non-instrumented).
#   profiles/capture.sh <tag> [bench args...]
set -e
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" > $OUT/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_knn --launch-skip 4 -c 1 \
  -o $OUT/k1_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" > $OUT/ncu_full.log 2>&1
echo done
