#!/bin/bash
# compute-sanitizer over every liboccx kernel (scripts/sanitize.py workload).
# racecheck runs once per kernel family so each gets its own hazard summary.
# Usage (repo root, under gpurun): bash scripts/sanitize.sh [tag]
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
KN="regex=score_|topk_merge|mix_reduce|feature_kernel|occ_dump|suggest_kernel|build_vtab|gen_space"
python scripts/sanitize.py > $OUT/sanitize_plain_$TAG.log 2>&1; echo "plain rc=$?"
for tool in memcheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  echo "compute-sanitizer --tool $tool $extra --kernel-name '$KN' python scripts/sanitize.py" > $OUT/sanitize_${tool}_$TAG.log
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --kernel-name "$KN" \
    python scripts/sanitize.py >> $OUT/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool rc=$?"; tail -1 $OUT/sanitize_${tool}_$TAG.log
done
for k in score_topk_tma score_topk_ldg score_space_kernel topk_merge mix_reduce feature_kernel \
         occ_dump suggest_kernel build_vtab gen_space; do
  log=$OUT/sanitize_racecheck_${k}_$TAG.log
  echo "compute-sanitizer --tool racecheck --racecheck-report all --kernel-name regex=$k python scripts/sanitize.py" > $log
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 \
    --kernel-name "regex=$k" python scripts/sanitize.py >> $log 2>&1
  echo "racecheck $k rc=$?: $(tail -1 $log)"
done
