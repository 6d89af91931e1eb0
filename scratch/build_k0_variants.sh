#!/bin/bash
# Build liboccx variants differing only in K0's OCCX_K0_LDS split (scratch/k0lib/).
set -e
cd "$(dirname "$0")/.."
O=paper_1701_08547_b200/_objs
for n in 0 2 4 6 8; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -cudart shared \
    -DOCCX_K0_LDS=$n -c paper_1701_08547_b200/csrc/occx_mix.cu -o /tmp/occx_mix_$n.o
  objs=$(ls $O/*.o | grep -v occx_mix.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared $objs /tmp/occx_mix_$n.o -o scratch/k0lib/liboccx_lds$n.so
done
ls -la scratch/k0lib
