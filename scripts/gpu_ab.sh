#!/bin/bash
# A/B of two library builds on one box: bash scripts/gpu_ab.sh VARIANT SCRIPT [rounds]
V=$1; S=$2; R=${3:-2}
for i in $(seq $R); do
  echo "== main"; timeout 300 python $S
  echo "== $V"; OCCX_LIB=paper_1701_08547_b200/_objs_$V/liboccx_$V.so timeout 300 python $S
done
