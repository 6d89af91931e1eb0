#!/bin/bash
TAG=${1:-r02n}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_abi_errors.py tests/test_gpu_parity.py tests/test_gpu_random.py -q -m gpu -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests_$TAG.log
python scripts/k2i_bench.py --every-key
python scripts/k2i_bench.py
python scripts/e2e_profile.py --every-key 2>&1 | tail -1
python scripts/k2_sizes.py 2>&1 | tail -3
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 5 --kernel-name "regex=score_topk_tma" python scripts/sanitize.py > $OUT/race_tma_$TAG.log 2>&1; tail -1 $OUT/race_tma_$TAG.log
