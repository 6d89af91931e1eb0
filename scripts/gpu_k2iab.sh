#!/bin/bash
timeout 900 python -m pytest tests -q -m gpu -x -k "k2i or implicit or score_space or space" 2>&1 | tail -1
for i in 1 2; do
  echo "== main"; timeout 300 python scripts/k2i_bench.py --every-key; timeout 300 python scripts/k2i_bench.py
  echo "== a"; OCCX_LIB=paper_1701_08547_b200/_objs_a/liboccx_a.so timeout 300 python scripts/k2i_bench.py --every-key; OCCX_LIB=paper_1701_08547_b200/_objs_a/liboccx_a.so timeout 300 python scripts/k2i_bench.py
done
