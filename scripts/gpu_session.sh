#!/bin/bash
# One GPU session: parity tests, smoke, bench (+reference arm), ncu evidence.
# Usage (from the repo root, under gpurun): bash scripts/gpu_session.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
timeout 1200 python -m pytest tests -q -m gpu > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref rc=$?"
# launch list of the bench command (cold, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
# full capture of the hot kernel on the bench workload, and of K2i (score_space path)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_topk -s 3 -c 1 -f \
  -o $OUT/k2_full_$TAG python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-secondary > /dev/null 2>&1; echo "ncu k2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_space_kernel -s 28 -c 1 -f \
  -o $OUT/k2i_full_$TAG python scripts/k2i_bench.py --every-key > /dev/null 2>&1; echo "ncu k2i rc=$?"
ls -la $OUT
