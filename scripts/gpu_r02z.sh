#!/bin/bash
# Refresh the K2i ncu capture after the range-max filter, then the bench line
# (its K2i issue roofline reads the committed capture's instruction count).
TAG=r02z
OUT=gpurun_out; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_space_kernel -s 28 -c 1 -f \
  -o $OUT/ncu_k2i_$TAG python scripts/k2i_bench.py --every-key > /dev/null 2>&1; echo "k2i rc=$?"
python scripts/ncu_digest.py $OUT/ncu_k2i_$TAG.ncu-rep $OUT/${TAG}_k2i_ncu --workload config5-1e9-orio-space --alg-bytes 0 --units 1284505600 --command "ncu --set full -k regex:score_space_kernel -s 28 -c 1 python scripts/k2i_bench.py --every-key" --note "K2i implicit grid, every key evaluated, runs filtered from range maxima; no candidate bytes in HBM"
cp $OUT/${TAG}_k2i_ncu.json profiles/r02_k2i_ncu_full.json
cp $OUT/${TAG}_k2i_ncu_ops.json profiles/r02_k2i_ncu_ops.json 2>/dev/null
cp $OUT/${TAG}_k2i_ncu_sass_top.csv profiles/r02_k2i_ncu_sass_top.csv 2>/dev/null
timeout 1200 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
