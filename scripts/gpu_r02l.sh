#!/bin/bash
TAG=${1:-r02l}
OUT=gpurun_out; mkdir -p $OUT
OCCX_LIB=paper_1701_08547_b200/_objs_timing/liboccx_timing.so timeout 600 python scripts/k2_profile.py config2 config4 shard8 config5 2>&1 | tee $OUT/k2_counts_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mix_reduce -s 2 -c 1 -f -o $OUT/k0_full_$TAG python scripts/ncu_workloads.py k0 > /dev/null 2>&1; echo "ncu k0 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_space_kernel -s 28 -c 1 -f -o $OUT/k2i_full_$TAG python scripts/k2i_bench.py --every-key > /dev/null 2>&1; echo "ncu k2i rc=$?"
