python scratch/k0_variants.py g > gpurun_out/k0_variants.log 2>&1
timeout 600 python -m pytest -x -q tests/test_gpu_random.py -k k0 tests/test_gpu_parity.py::test_k0_full_corpus_vs_oracle tests/test_gpu_parity.py::test_k0_corpus_golden tests/test_gpu_parity.py::test_tokenizer_plus_k0_corpus_golden tests/test_gpu_parity.py::test_k0_atax_fixture > gpurun_out/k0_tests.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mix_reduce -s 3 -c 1 -o gpurun_out/k0_full_g python scratch/k0_variants.py g > /dev/null 2>&1
cat gpurun_out/k0_variants.log; tail -5 gpurun_out/k0_tests.log
