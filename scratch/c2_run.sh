#!/bin/bash
# config-2/4 K2 split + one ncu full capture of config-2 K2
mkdir -p gpurun_out
python scratch/c2_parts.py config2 config4 > gpurun_out/c2_parts.log 2>&1; echo parts rc=$?; cat gpurun_out/c2_parts.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_list.csv python scratch/c2_parts.py config2 > /dev/null 2>&1; echo list rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_topk -s 5 -c 1 -f -o gpurun_out/c2_k2 python scratch/c2_parts.py config2 > /dev/null 2>&1; echo full rc=$?
