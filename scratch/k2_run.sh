#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_random.py tests/test_gpu_parity.py -k "k2 or score or config or shard" > gpurun_out/k2_tests.log 2>&1; tail -3 gpurun_out/k2_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-secondary --no-e2e > gpurun_out/k2_bench.json 2>gpurun_out/k2_bench.err; python -c "
import json; d=json.load(open('gpurun_out/k2_bench.json')); print(d['value']/1e9, d['roofline']['kernel_ms'], d['roofline']['frac'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_topk -s 3 -c 1 -f -o gpurun_out/k2_full python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-secondary > /dev/null 2>&1
