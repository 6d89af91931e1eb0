#!/bin/bash
# GPU tests, K2 per-call-size timing (plain + instrumented build), per-kernel racecheck.
TAG=${1:-r02b}
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests_$TAG.log
timeout 600 python scripts/k2_profile.py > $OUT/k2_profile_$TAG.log 2>&1; echo "k2 profile rc=$?"; cat $OUT/k2_profile_$TAG.log
OCCX_LIB=paper_1701_08547_b200/_objs_timing/liboccx_timing.so timeout 600 python scripts/k2_profile.py > $OUT/k2_profile_timing_$TAG.log 2>&1; echo "k2 timing rc=$?"; cat $OUT/k2_profile_timing_$TAG.log
timeout 2400 bash scripts/sanitize.sh $TAG
