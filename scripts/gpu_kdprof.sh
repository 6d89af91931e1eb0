#!/bin/bash
TAG=${1:-kd}
OUT=gpurun_out; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:occ_dump -s 2 -c 1 -f \
  -o $OUT/${TAG} python scripts/ncu_workloads.py kd > /dev/null 2>&1; echo "ncu rc=$?"
ncu -i $OUT/${TAG}.ncu-rep --page source --csv --print-source sass > $OUT/${TAG}_sass.csv 2>/dev/null; echo "src rc=$?"
python scripts/ncu_digest.py $OUT/${TAG}.ncu-rep $OUT/${TAG}_ncu --workload acceptance-7a-sweep --alg-bytes 77070336 --units 1605632 --command "ncu --set full -k regex:occ_dump -s 2 -c 1 python scripts/ncu_workloads.py kd" --note "Kd"
