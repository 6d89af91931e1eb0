#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_random.py tests/test_gpu_parity.py -k "k2i or score_space or implicit or shard" > gpurun_out/k2i_tests.log 2>&1; tail -3 gpurun_out/k2i_tests.log
python scripts/k2i_bench.py > gpurun_out/k2i_bench.log 2>&1; cat gpurun_out/k2i_bench.log
python scratch/api_profile.py > gpurun_out/api_profile.log 2>&1; tail -2 gpurun_out/api_profile.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_space_kernel -s 28 -c 1 -f -o gpurun_out/k2i_full python scripts/k2i_bench.py > /dev/null 2>&1
