#!/bin/bash
# Round-end evidence session: GPU tests, smoke, bench (both arms), launch
# list, ncu --set full of every kernel family, compute-sanitizer.
# Usage (repo root, under gpurun): bash scripts/gpu_evidence.sh TAG
TAG=${1:-r02}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu_$TAG.txt
timeout 1200 python -m pytest tests -q -m gpu -rs > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gpu_tests_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
timeout 1200 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-secondary > /dev/null 2>&1; echo "ncu list rc=$?"
N="ncu --set full --clock-control none --import-source on -f"
timeout 900 $N -k regex:score_topk_tma -s 3 -c 1 -o $OUT/ncu_k2_$TAG python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-secondary > /dev/null 2>&1; echo "k2 rc=$?"
timeout 600 $N -k regex:score_space_kernel -s 28 -c 1 -o $OUT/ncu_k2i_$TAG python scripts/k2i_bench.py --every-key > /dev/null 2>&1; echo "k2i rc=$?"
for w in k0 kd k1 k3 k4; do
  case $w in k0) K=mix_reduce;; kd) K=occ_dump;; k1) K=feature_kernel;; k3) K=topk_merge;; k4) K=suggest_kernel;; esac
  timeout 600 $N -k regex:$K -s 2 -c 1 -o $OUT/ncu_${w}_$TAG python scripts/ncu_workloads.py $w > /dev/null 2>&1; echo "$w rc=$?"
done
# digest the reports on the box (gpurun copies back <= 64 MiB)
D="python scripts/ncu_digest.py"
$D $OUT/ncu_k2_$TAG.ncu-rep $OUT/${TAG}_k2_ncu --workload config5-1e9-orio-space --alg-bytes 20552089600 --units 1284505600 --command "ncu --set full -k regex:score_topk_tma -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-secondary" --note "K2 record scorer, config 5, one GPU"
$D $OUT/ncu_k2i_$TAG.ncu-rep $OUT/${TAG}_k2i_ncu --workload config5-1e9-orio-space --alg-bytes 0 --units 1284505600 --command "ncu --set full -k regex:score_space_kernel -s 28 -c 1 python scripts/k2i_bench.py --every-key" --note "K2i implicit grid, every key evaluated; no candidate bytes in HBM"
$D $OUT/ncu_k0_$TAG.ncu-rep $OUT/${TAG}_k0_ncu --workload config3-100k-kernel-sass-corpus --alg-bytes 424898800 --units 102424698 --command "ncu --set full -k regex:mix_reduce -s 2 -c 1 python scripts/ncu_workloads.py k0" --note "K0 on class records (identity class table)"
$D $OUT/ncu_kd_$TAG.ncu-rep $OUT/${TAG}_kd_ncu --workload acceptance-7a-sweep --alg-bytes 77070336 --units 1605632 --command "ncu --set full -k regex:occ_dump -s 2 -c 1 python scripts/ncu_workloads.py kd" --note "Kd: 16 B in + 32 B out per launch"
$D $OUT/ncu_k1_$TAG.ncu-rep $OUT/${TAG}_k1_ncu --workload config3-corpus-mixes-x4 --alg-bytes 115200000 --units 400000 --command "ncu --set full -k regex:feature_kernel -s 2 -c 1 python scripts/ncu_workloads.py k1" --note "K1: 144 B mix in, 240 B features out per (mix, column), 48 B sums per mix"
$D $OUT/ncu_k3_$TAG.ncu-rep $OUT/${TAG}_k3_ncu --workload config5-partials --alg-bytes 381440 --units 20 --command "ncu --set full -k regex:topk_merge -s 2 -c 1 python scripts/ncu_workloads.py k3" --note "K3: 148 tables x 20 segments x 16 keys in, 20 x 16 out"
$D $OUT/ncu_k4_$TAG.ncu-rep $OUT/${TAG}_k4_ncu --workload suggest-100k-kernels-x5-archs --alg-bytes 24000000 --units 500000 --command "ncu --set full -k regex:suggest_kernel -s 2 -c 1 python scripts/ncu_workloads.py k4" --note "K4: 16 B request in, 32 B result out"
du -sh $OUT
timeout 2400 bash scripts/sanitize.sh $TAG
ls $OUT | grep $TAG
