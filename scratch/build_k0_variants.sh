#!/bin/bash
# Build liboccx variants differing only in K0 compile-time knobs (scratch/k0lib/); the
# THREADS/CTAS/DEPTH knobs were experiment-only (reverted), LDS is OCCX_K0_LDS:
#   OCCX_K0_LDS (table vs arithmetic increments); the register-feed experiment was reverted
set -e
cd "$(dirname "$0")/.."
O=paper_1701_08547_b200/_objs
mkdir -p scratch/k0lib
for v in "$@"; do            # v = THREADS:CTAS:LDS
  IFS=: read t c l d <<< "$v"; d=${d:-4}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -cudart shared \
    -DOCCX_K0_LDS=$l -DOCCX_K0_THREADS=$t -DOCCX_K0_CTAS=$c -DOCCX_K0_DEPTH=$d -Xptxas -v -c paper_1701_08547_b200/csrc/occx_mix.cu -o /tmp/occx_mix_v.o 2>&1 | grep -A2 "ILi4" | grep -i "registers\|spill" | sed "s/^/T$t C$c L$l /"
  objs=$(ls $O/*.o | grep -v occx_mix.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared $objs /tmp/occx_mix_v.o -o scratch/k0lib/liboccx_t${t}_c${c}_l${l}_d${d}.so
done
