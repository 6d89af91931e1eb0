timeout 600 python -m pytest tests -q -m gpu -x -k "k0 or tokenizer or mix or aggregate or ragged or csr" 2>&1 | tail -3
timeout 300 python scripts/k0_time.py
