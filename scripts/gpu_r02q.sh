#!/bin/bash
echo "== default"; timeout 300 python scripts/k2_sizes.py
echo "== stream-only (no scoring)"; OCCX_LIB=paper_1701_08547_b200/_objs_stream/liboccx_stream.so timeout 300 python scripts/k2_sizes.py
echo "== stream-only, no steal"; K2_OPTIONS=4 OCCX_LIB=paper_1701_08547_b200/_objs_stream/liboccx_stream.so timeout 300 python scripts/k2_sizes.py
echo "== stream-only, one slice"; K2_OPTIONS=2 OCCX_LIB=paper_1701_08547_b200/_objs_stream/liboccx_stream.so timeout 300 python scripts/k2_sizes.py
