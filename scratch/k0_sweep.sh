#!/bin/bash
mkdir -p gpurun_out
for n in 0 2 4 6 8; do
  OCCX_LIB=scratch/k0lib/liboccx_lds$n.so python scratch/k0_variants.py g 2>&1 | sed "s/^/lds=$n /"
done | tee gpurun_out/k0_sweep.log
OCCX_LIB=scratch/k0lib/liboccx_lds4.so timeout 600 python -m pytest -x -q tests/test_gpu_random.py tests/test_gpu_parity.py -k "k0 or ragged or corpus or atax" 2>&1 | tail -2
