#!/bin/bash
# K0 A/B against a named variant build: bash scripts/gpu_k0v.sh VARIANT
timeout 600 env OCCX_LIB=paper_1701_08547_b200/_objs_$1/liboccx_$1.so python -m pytest tests -q -m gpu -x -k "k0 or mix or aggregate" 2>&1 | tail -1
bash scripts/gpu_ab.sh $1 scripts/k0_time.py 2
