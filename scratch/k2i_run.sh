#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_random.py tests/test_gpu_parity.py -k "k2i or score_space or implicit" > gpurun_out/k2i_tests.log 2>&1; tail -5 gpurun_out/k2i_tests.log
python scratch/k2i_bench.py > gpurun_out/k2i_bench.log 2>&1; cat gpurun_out/k2i_bench.log
python scratch/api_profile.py > gpurun_out/api_profile.log 2>&1; tail -60 gpurun_out/api_profile.log | head -70
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_space_kernel -s 28 -c 1 -f -o gpurun_out/k2i_full python scratch/k2i_bench.py > /dev/null 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-secondary > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; cat gpurun_out/bench_quick.json; tail -3 gpurun_out/bench_quick.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --workload config4 --no-cpu > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; cat gpurun_out/bench_gloo2.json; tail -5 gpurun_out/bench_gloo2.err
