#!/bin/bash
TAG=${1:-r02c}
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests_$TAG.log
timeout 600 python scripts/k2_profile.py > $OUT/k2_profile_$TAG.log 2>&1; echo "k2 profile rc=$?"; cat $OUT/k2_profile_$TAG.log
OCCX_LIB=paper_1701_08547_b200/_objs_timing/liboccx_timing.so timeout 600 python scripts/k2_profile.py > $OUT/k2_profile_timing_$TAG.log 2>&1; echo "k2 timing rc=$?"; cat $OUT/k2_profile_timing_$TAG.log
timeout 900 python bench.py --no-cpu --no-secondary > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; tail -c 1500 $OUT/bench_$TAG.json
timeout 600 compute-sanitizer --tool initcheck --kernel-name "regex=mix_reduce|score_topk" python scripts/sanitize.py > $OUT/sanitize_initcheck_$TAG.log 2>&1; echo "initcheck: $(tail -1 $OUT/sanitize_initcheck_$TAG.log)"
