#!/bin/bash
# Build liboccx variants differing only in K0 compile-time knobs (scratch/k0lib/):
#   OCCX_K0_LDS (table vs arithmetic increments); the register-feed experiment was reverted
set -e
cd "$(dirname "$0")/.."
O=paper_1701_08547_b200/_objs
mkdir -p scratch/k0lib
for v in "$@"; do            # v = FEED:LDS
  f=${v%%:*}; l=${v##*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -cudart shared \
    -DOCCX_K0_LDS=$l -DOCCX_K0_FEED=$f -Xptxas -v -c paper_1701_08547_b200/csrc/occx_mix.cu -o /tmp/occx_mix_$f_$l.o 2>&1 | grep -A2 "ILi4" | grep -i "registers\|spill" | sed "s/^/F$f L$l /"
  objs=$(ls $O/*.o | grep -v occx_mix.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared $objs /tmp/occx_mix_$f_$l.o -o scratch/k0lib/liboccx_f${f}_l${l}.so
done
