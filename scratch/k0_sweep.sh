#!/bin/bash
mkdir -p gpurun_out
for f in scratch/k0lib/liboccx_*.so; do
  OCCX_LIB=$f python scratch/k0_variants.py g 2>&1 | sed "s#^#$(basename $f) #"
done | tee gpurun_out/k0_sweep.log
