#!/bin/bash
# compute-sanitizer over every liboccx kernel (scripts/sanitize.py workload).
# Usage (repo root, under gpurun): bash scripts/sanitize.sh [tag]
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
KN="regex=score_|topk_merge|mix_reduce|feature_kernel|occ_dump|suggest_kernel|build_vtab|gen_space"
python scripts/sanitize.py > $OUT/sanitize_plain_$TAG.log 2>&1; echo "plain rc=$?"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  [ $tool = memcheck ] && extra="--leak-check no"
  echo "compute-sanitizer --tool $tool $extra --kernel-name '$KN' python scripts/sanitize.py" > $OUT/sanitize_${tool}_$TAG.log
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --kernel-name "$KN" \
    python scripts/sanitize.py >> $OUT/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool rc=$?"; tail -3 $OUT/sanitize_${tool}_$TAG.log
done
