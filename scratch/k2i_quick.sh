#!/bin/bash
timeout 900 python -m pytest -x -q tests/test_gpu_random.py tests/test_gpu_parity.py -k "k2i or implicit or score_space" 2>&1 | tail -1
python scripts/k2i_bench.py
