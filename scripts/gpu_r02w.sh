#!/bin/bash
# Final round-2 check on the shipped library: GPU tests, smoke, bench (both arms).
TAG=${1:-r02w}
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -rs > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
timeout 1200 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 600 python bench.py --gpus 2 --dist-backend gloo --steps 3 --warmup 3 --no-cpu --no-e2e > $OUT/bench_gloo2_$TAG.json 2> $OUT/bench_gloo2_$TAG.err; echo "gloo2 rc=$?"; tail -c 600 $OUT/bench_gloo2_$TAG.json
