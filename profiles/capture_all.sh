#!/bin/bash
# ncu --set full of every kernel the BASELINE paths launch (one representative full-size launch
# each), run on a GPU box from the repo root.  Reports land in gpurun_out/<tag>/; digest them with
#   python profiles/ncu_digest.py gpurun_out/<tag>/*.ncu-rep --md
#   profiles/capture_all.sh <tag>
TAG=$1
OUT=gpurun_out/$TAG
mkdir -p $OUT
python profiles/ncu_drive.py c2 > $OUT/drive_c2.log 2>&1 || { echo "c2 drive failed"; exit 1; }
python profiles/ncu_drive.py c5 > $OUT/drive_c5.log 2>&1 || { echo "c5 drive failed"; exit 1; }
cap() {  # <name> <what> <kernel regex> <launch-skip>
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$3" --launch-skip $4 -c 1 \
    -o $OUT/$1 python profiles/ncu_drive.py $2 > $OUT/$1.log 2>&1 || echo "capture $1 failed"
}
cap k1_c2 c2 'k_knn<' 0
cap build0_c2 c2 'k_build<3, 0>' 0
cap build1_c2 c2 'k_build<3, 1>' 0
cap slotrank_c2 c2 'k_slot_rank' 0
cap emit_c2 c2 'k_emit' 0
cap qbox_c2 c2 'k_qbox<' 0
cap curvekey_c2 c2 'k_curve_key' 0
cap onesweep_c2 c2 'Onesweep' 0
cap range2_c2 c2 'k_range<3, 2>' 0
cap range1_c2 c2 'k_range<3, 1>' 0
cap slotscompact_c2 c2 'k_slots_compact' 0
cap ingest_c2 c2 'k_ingest' 0
cap erase_c5 c5 'k_erase' 0
cap bloom_c5 c5 'k_bloom_build' 0
cap collapse_c5 c5 'k_collapse_up' 0
cap relink_c5 c5 'k_relink' 0
cap k1_c5 c5 'k_knn<' 0
echo capture_all done
