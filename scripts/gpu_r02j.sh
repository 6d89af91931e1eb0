#!/bin/bash
TAG=${1:-r02j}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gpu_tests_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python scripts/e2e_profile.py --every-key 2>&1 | tail -2
timeout 300 python scripts/e2e_profile.py 2>&1 | tail -2
timeout 900 python bench.py --no-cpu --no-secondary > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; tail -2 $OUT/bench_$TAG.err
python -c "
import json;d=json.loads(open('$OUT/bench_$TAG.json').read().strip().splitlines()[-1]); print('value',d['value'],'ms',d['ms_per_step']); print('e2e',d['e2e'].get('value'), d['e2e'].get('ms_per_step'), 'pruned', d['e2e'].get('pruned'))"
