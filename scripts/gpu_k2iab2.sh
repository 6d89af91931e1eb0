#!/bin/bash
timeout 900 python -m pytest tests -q -m gpu -x -k "k2i or implicit or score_space or space" 2>&1 | tail -1
for i in 1 2; do
  echo "== main"; timeout 300 python scripts/k2i_bench.py --every-key | grep K2i; timeout 300 python scripts/k2i_bench.py | grep K2i
  echo "== b"; OCCX_LIB=paper_1701_08547_b200/_objs_b/liboccx_b.so timeout 300 python scripts/k2i_bench.py --every-key | grep K2i; OCCX_LIB=paper_1701_08547_b200/_objs_b/liboccx_b.so timeout 300 python scripts/k2i_bench.py | grep K2i
done
