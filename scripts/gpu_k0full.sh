#!/bin/bash
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python scripts/k0_time.py
