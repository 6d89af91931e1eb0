#!/bin/bash
TAG=${1:-r02f}
OUT=gpurun_out
mkdir -p $OUT
for opt in 0 4; do
  K2_OPTIONS=$opt timeout 600 python scripts/k2_profile.py > $OUT/k2_profile_o${opt}_$TAG.log 2>&1; echo "k2 options=$opt rc=$?"; cat $OUT/k2_profile_o${opt}_$TAG.log
done
timeout 300 python scripts/e2e_profile.py --every-key > $OUT/e2e_prof_$TAG.log 2>&1; cat $OUT/e2e_prof_$TAG.log | head -40
timeout 300 python scripts/e2e_profile.py > $OUT/e2e_prof_pruned_$TAG.log 2>&1; head -3 $OUT/e2e_prof_pruned_$TAG.log
