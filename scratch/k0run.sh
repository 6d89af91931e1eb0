#!/bin/bash
# K0 iteration: parity tests, timing (L2 flushed), one full ncu capture with source.
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q tests/test_gpu_random.py tests/test_gpu_parity.py tests/test_gpu_report.py -k "k0 or ragged or report or corpus or atax" > gpurun_out/k0_tests.log 2>&1
tail -3 gpurun_out/k0_tests.log
python scratch/k0_variants.py g > gpurun_out/k0_variants.log 2>&1
cat gpurun_out/k0_variants.log
if [ "${NCU:-1}" = 1 ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mix_reduce -s 3 -c 1 -f -o gpurun_out/k0_full_g python scratch/k0_variants.py g > /dev/null 2>&1
fi
