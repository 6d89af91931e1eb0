#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
for g in 0 1; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_topk_tma -s 2 -c 1 -f \
  -o $OUT/k2_shard${g}_r02i python scripts/k2_one_shard.py $g 8 > $OUT/ncu_shard${g}.log 2>&1; echo "ncu shard $g rc=$?"
done
