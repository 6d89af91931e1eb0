"""Tokenizer stage times on the 1000-kernel config-3 listing:
python scripts/tok_breakdown.py"""
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1701_08547_b200 import _lib, sass  # noqa: E402
from paper_1701_08547_b200.mix import DEFAULT_OPCLASSES  # noqa: E402

text = "".join(bench._corpus_text_part((k, min(k + 100, 1000))) for k in range(0, 1000, 100))
lines = text.count("\n")
lib = _lib.load()
print(f"{lines} lines, {len(text) / 1e6:.1f} MB, {os.cpu_count()} cpus, affinity {len(os.sched_getaffinity(0))}")


def med(fn, n=5):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


data = text.encode("utf-8", "surrogatepass")
print(f"encode {med(lambda: text.encode('utf-8', 'surrogatepass')):.1f} ms")
for chunk in (0, 1 << 30, 4 << 20, 256 << 10):
    def parse():
        h = ctypes.c_void_p()
        line = ctypes.c_int64(0)
        lib.occx_sass_parse_ex(data, len(data), chunk, ctypes.byref(h), ctypes.byref(line))
        lib.occx_sass_free(h)
    print(f"native parse chunk={chunk}: {med(parse):.1f} ms")
print(f"tokenize(table) {med(lambda: sass.tokenize(text, table=DEFAULT_OPCLASSES)):.1f} ms")
print(f"tokenize() {med(lambda: sass.tokenize(text)):.1f} ms")
r = sass.tokenize(text)
print(f"class_lut {med(lambda: r.class_lut(DEFAULT_OPCLASSES)):.1f} ms")
print(f"aggregate_text {med(lambda: sass.aggregate_text(text)):.1f} ms")
