#!/bin/bash
# Kd CTA-shape sweep (experiment builds via OCCX_LIB)
echo "== main (256 x 8, 32 regs)"; timeout 300 python scripts/kd_time.py
for v in kd256 kd512 kd1024 a; do echo "== $v"; OCCX_LIB=paper_1701_08547_b200/_objs_$v/liboccx_$v.so timeout 300 python scripts/kd_time.py; done
