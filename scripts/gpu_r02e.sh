#!/bin/bash
TAG=${1:-r02e}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_abi_errors.py tests/test_gpu_parity.py tests/test_gpu_random.py -q -m gpu -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests_$TAG.log
for opt in 0 4; do
  K2_OPTIONS=$opt timeout 600 python scripts/k2_profile.py > $OUT/k2_profile_o${opt}_$TAG.log 2>&1; echo "k2 options=$opt rc=$?"; cat $OUT/k2_profile_o${opt}_$TAG.log
done
OCCX_LIB=paper_1701_08547_b200/_objs_timing/liboccx_timing.so timeout 600 python scripts/k2_profile.py shard8 config2 > $OUT/k2_profile_timing_$TAG.log 2>&1; cat $OUT/k2_profile_timing_$TAG.log
timeout 300 python scripts/k2i_bench.py --every-key > $OUT/k2i_$TAG.log 2>&1; cat $OUT/k2i_$TAG.log
timeout 300 python scripts/k2i_bench.py > $OUT/k2i_pruned_$TAG.log 2>&1; cat $OUT/k2i_pruned_$TAG.log
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 5 --kernel-name "regex=score_space|score_topk_ldg" python scripts/sanitize.py > $OUT/race_$TAG.log 2>&1; tail -1 $OUT/race_$TAG.log
