#!/bin/bash
# K0 work-split weight sweep (experiment builds via OCCX_LIB)
echo "kw 512 (default)"; timeout 300 python scripts/k0_time.py
for kw in 256 1024 2048; do echo "kw $kw"; OCCX_LIB=paper_1701_08547_b200/_objs_kw$kw/liboccx_kw$kw.so timeout 300 python scripts/k0_time.py; done
