#!/bin/bash
echo "== default (16 consumer warps)"; timeout 300 python scripts/k2_sizes.py 2>&1 | tail -5
echo "== 24 consumer warps"; OCCX_LIB=paper_1701_08547_b200/_objs_c24/liboccx_c24.so timeout 300 python scripts/k2_sizes.py 2>&1 | tail -5
OCCX_LIB=paper_1701_08547_b200/_objs_c24/liboccx_c24.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "k2 or config" 2>&1 | tail -1
