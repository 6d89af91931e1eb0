#!/bin/bash
TAG=${1:-r02u}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
python - <<PY
import json
d=json.loads(open("$OUT/bench_$TAG.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value","ms_per_step")}, d["roofline"]["frac"], d["e2e"]["value"], d["e2e"]["ms_per_step"])
for k,v in d["secondary"].items():
    print(k, json.dumps(v)[:700])
PY
