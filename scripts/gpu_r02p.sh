#!/bin/bash
for lib in "" paper_1701_08547_b200/_objs_f64/liboccx_f64.so; do
  for opt in 0 4; do
    echo "== lib=${lib:-default} options=$opt"
    OCCX_LIB=$lib K2_OPTIONS=$opt timeout 300 python scripts/k2_sizes.py 2>&1 | tail -4
  done
done
OCCX_LIB= timeout 300 python scripts/k2_shards.py
OCCX_LIB=paper_1701_08547_b200/_objs_f64/liboccx_f64.so timeout 300 python scripts/k2_shards.py
