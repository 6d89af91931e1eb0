#!/bin/bash
# Evidence after the K0 rework: tests, smoke, bench (both arms), launch list,
# K0 ncu --set full (+ SASS source page), K0 sanitizer runs.
TAG=${1:-r02v}
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -rs > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
timeout 1200 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
N="ncu --set full --clock-control none --import-source on -f"
timeout 600 $N -k regex:mix_reduce -s 2 -c 1 -o $OUT/ncu_k0_$TAG python scripts/ncu_workloads.py k0 > /dev/null 2>&1; echo "k0 rc=$?"
ncu -i $OUT/ncu_k0_$TAG.ncu-rep --page source --csv --print-source sass > $OUT/${TAG}_k0_sass.csv 2>/dev/null
python scripts/ncu_digest.py $OUT/ncu_k0_$TAG.ncu-rep $OUT/${TAG}_k0_ncu --workload config3-100k-kernel-sass-corpus --alg-bytes 424898800 --units 102424698 --command "ncu --set full -k regex:mix_reduce -s 2 -c 1 python scripts/ncu_workloads.py k0" --note "K0 on class records (identity class table)"
python scripts/sanitize.py > $OUT/sanitize_plain_$TAG.log 2>&1; echo "plain rc=$?"
for tool in memcheck synccheck initcheck; do
  echo "compute-sanitizer --tool $tool --kernel-name regex=mix_reduce python scripts/sanitize.py" > $OUT/sanitize_${tool}_mix_reduce_$TAG.log
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --kernel-name "regex=mix_reduce" \
    python scripts/sanitize.py >> $OUT/sanitize_${tool}_mix_reduce_$TAG.log 2>&1
  echo "$tool rc=$?: $(tail -1 $OUT/sanitize_${tool}_mix_reduce_$TAG.log)"
done
log=$OUT/sanitize_racecheck_mix_reduce_$TAG.log
echo "compute-sanitizer --tool racecheck --racecheck-report all --kernel-name regex=mix_reduce python scripts/sanitize.py" > $log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 --kernel-name "regex=mix_reduce" python scripts/sanitize.py >> $log 2>&1
echo "racecheck rc=$?: $(tail -1 $log)"
ls $OUT | grep $TAG
