#!/bin/bash
TAG=${1:-r02r}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py -q -m gpu -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests_$TAG.log
timeout 300 python scripts/k2i_bench.py --every-key
timeout 300 python scripts/k2i_bench.py
timeout 300 python scripts/e2e_profile.py --every-key 2>&1 | tail -1
timeout 300 python scripts/e2e_profile.py 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_space_kernel -s 28 -c 1 -f -o $OUT/k2i_$TAG python scripts/k2i_bench.py --every-key > /dev/null 2>&1
python scripts/ncu_digest.py $OUT/k2i_$TAG.ncu-rep $OUT/${TAG}_k2i_ncu --workload config5-1e9-orio-space --alg-bytes 0 --units 1284505600 --command "ncu --set full -k regex:score_space_kernel -s 28 -c 1 python scripts/k2i_bench.py --every-key" --note "K2i, packed 16-bit inner loop"
python -c "import json; d=json.load(open('$OUT/${TAG}_k2i_ncu.json')); print({k: d[k] for k in ('duration_ms','issue_active_pct','alu_pipe_pct','warp_instructions','thread_instructions_per_unit','smem_bank_conflicts','smem_wavefronts')})"
