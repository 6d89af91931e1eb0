#!/bin/bash
# Re-entry check: smoke, full GPU tests, bench (both arms) on the rebuilt library.
TAG=${1:-r02t}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; cut -c1-400 $OUT/bench_$TAG.json
timeout 900 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref rc=$?"; cut -c1-300 $OUT/bench_ref_$TAG.json
