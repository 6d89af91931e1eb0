#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_space_kernel -s 28 -c 1 -f -o gpurun_out/k2i_full python scripts/k2i_bench.py > /dev/null 2>&1
ls -la gpurun_out/k2i_full.ncu-rep
