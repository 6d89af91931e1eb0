#!/bin/bash
# K0 ncu capture on config 3 (class records): full set + SASS source page
TAG=${1:-k0}
OUT=gpurun_out; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mix_reduce -s 2 -c 1 -f \
  -o $OUT/${TAG} python scripts/ncu_workloads.py k0 > /dev/null 2>&1; echo "ncu rc=$?"
ncu -i $OUT/${TAG}.ncu-rep --page source --csv --print-source sass > $OUT/${TAG}_sass.csv 2>/dev/null; echo "src rc=$?"
python scripts/ncu_digest.py $OUT/${TAG}.ncu-rep $OUT/${TAG}_ncu --workload config3-100k-kernel-sass-corpus \
  --alg-bytes 424898800 --units 102424698 --command "ncu --set full -k regex:mix_reduce -s 2 -c 1 python scripts/ncu_workloads.py k0" \
  --note "K0 on class records" --keep
ls -la $OUT
