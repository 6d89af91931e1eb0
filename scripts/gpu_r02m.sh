#!/bin/bash
TAG=${1:-r02m}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_abi_errors.py tests/test_gpu_parity.py -q -m gpu -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests_$TAG.log
python scripts/k2_sizes.py 2>&1 | tail -4
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 5 --kernel-name "regex=score_topk_tma" python scripts/sanitize.py > $OUT/race_tma_$TAG.log 2>&1; tail -1 $OUT/race_tma_$TAG.log
