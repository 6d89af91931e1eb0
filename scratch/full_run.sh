#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q tests -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python scratch/k2i_bench.py > gpurun_out/k2i_bench.log 2>&1; cat gpurun_out/k2i_bench.log
python scratch/api_profile.py > gpurun_out/api_profile.log 2>&1; tail -3 gpurun_out/api_profile.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-secondary > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; python -c "
import json; d=json.load(open('gpurun_out/bench_quick.json')); print(d['value']/1e9, d['e2e'], d.get('e2e_records',{}).get('value'))"; tail -3 gpurun_out/bench_quick.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --workload config4 --no-cpu > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; cat gpurun_out/bench_gloo2.json; grep -i "error" gpurun_out/bench_gloo2.err | head -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --workload config4 --scaling strong --no-cpu > gpurun_out/bench_gloo2s.json 2> gpurun_out/bench_gloo2s.err; cat gpurun_out/bench_gloo2s.json; grep -i "error" gpurun_out/bench_gloo2s.err | head -5
