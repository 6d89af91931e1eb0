#!/bin/bash
TAG=${1:-r02k}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_abi_errors.py -q -m gpu -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests_$TAG.log
python scripts/k2_sizes.py
python scripts/k2_shards.py
K2_OPTIONS=4 python scripts/k2_shards.py
python scripts/k2i_bench.py --every-key
