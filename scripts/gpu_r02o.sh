#!/bin/bash
TAG=${1:-r02o}
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/k2i_bench.py --every-key
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_space_kernel -s 28 -c 1 -f -o $OUT/k2i_full_$TAG python scripts/k2i_bench.py --every-key > /dev/null 2>&1; echo "ncu k2i rc=$?"
