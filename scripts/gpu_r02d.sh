#!/bin/bash
TAG=${1:-r02d}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_abi_errors.py tests/test_gpu_parity.py -q -m gpu -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests_$TAG.log
for opt in 0 4 8; do
  K2_OPTIONS=$opt timeout 600 python scripts/k2_profile.py > $OUT/k2_profile_o${opt}_$TAG.log 2>&1; echo "k2 options=$opt rc=$?"; cat $OUT/k2_profile_o${opt}_$TAG.log
done
K2_OPTIONS=4 OCCX_LIB=paper_1701_08547_b200/_objs_timing/liboccx_timing.so timeout 600 python scripts/k2_profile.py shard8 config5 > $OUT/k2_profile_timing_o4_$TAG.log 2>&1; cat $OUT/k2_profile_timing_o4_$TAG.log
timeout 1500 python bench.py --no-e2e > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; tail -3 $OUT/bench_$TAG.err
