#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_random.py tests/test_gpu_parity.py -k "k2 or score or config or shard" > gpurun_out/k2_tests.log 2>&1; tail -2 gpurun_out/k2_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/k2_bench.json 2>gpurun_out/k2_bench.err; python -c "
import json; d=json.load(open('gpurun_out/k2_bench.json')); s=d['secondary']; print(d['value']/1e9, d['roofline']['kernel_ms'], d['roofline']['frac']); print({k: (round(v.get('value',0)/1e9,1), v.get('ms'), v.get('roofline',{}).get('frac')) for k,v in s.items()})"
tail -2 gpurun_out/k2_bench.err
