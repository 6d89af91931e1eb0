"""Tokenizer and config-3 text e2e (bench.py secondary_config3_e2e):
python scripts/tok_time.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

r = bench.secondary_config3_e2e()
print(json.dumps({k: r[k] for k in ("workload", "e2e", "tokenizer")}))
print("cpu", r["cpu_baseline"]["value"], r["cpu_baseline"]["lines_per_s_parse"])
