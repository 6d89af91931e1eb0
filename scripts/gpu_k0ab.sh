#!/bin/bash
timeout 600 python -m pytest tests -q -m gpu -x -k "k0 or tokenizer or mix or aggregate" 2>&1 | tail -2
bash scripts/gpu_ab.sh a scripts/k0_time.py 2
