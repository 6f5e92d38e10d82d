#!/bin/bash
# final round-2 measurements on the GPU box: GPU tests, bench lines (both arms), launch list of the bench
# command, ncu --set full digests of the kernels of the BASELINE paths, K1 traffic JSON for bench.py
OUT=gpurun_out/r2z
mkdir -p $OUT
python -m pytest tests -m gpu -x -q > $OUT/gputest.log 2>&1; tail -2 $OUT/gputest.log
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras --no-configs > $OUT/ncu_launch.log 2>&1
bash profiles/capture_some.sh r2z "k1_c2 c2 k_knn<" "build0_c2 c2 k_build<.int.3,_SP_.int.0>" "subtree_c2 c2 k_subtree" \
  "merge_c2 c2 k_merge" "emit_c2 c2 k_emit" "erase_c5 c5 k_erase" "build0_c5 c5 k_build<.int.2,_SP_.int.0>" \
  "subtree_c5 c5 k_subtree" > $OUT/capture.log 2>&1
python profiles/ncu_digest.py /tmp/ncu_k1_c2.ncu-rep --k1-json $OUT/k1_traffic.json --config 2 > $OUT/k1_digest.txt 2>&1
tail -c 300 $OUT/bench.json
