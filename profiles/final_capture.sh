#!/bin/bash
# final round-2 measurements: bench lines, launch list of the bench command, ncu --set full digests
OUT=gpurun_out/r2f
mkdir -p $OUT
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras --no-configs > $OUT/ncu_launch.log 2>&1
bash profiles/capture_some.sh r2f "k1_c2 c2 k_knn<" "build0_c2 c2 k_build<3,_SP_0>" "build1_c2 c2 k_build<3,_SP_1>" \
  "subtree_c2 c2 k_subtree" "merge_c2 c2 k_merge" "emit_c2 c2 k_emit" "erase_c5 c5 k_erase" "collapse_c5 c5 k_collapse_up" \
  "bloom_c5 c5 k_bloom_build" "k1_c5 c5 k_knn<" "build0_c5 c5 k_build<2,_SP_0>" "k1_c3 c3 k_knn<" > $OUT/capture.log 2>&1
python profiles/ncu_digest.py /tmp/ncu_k1_c2.ncu-rep --k1-json $OUT/k1_traffic.json --config 2 > $OUT/k1_digest.txt 2>&1
tail -c 300 $OUT/bench.json
