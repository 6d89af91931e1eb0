"""K0 time on config 3 (class records and signature records), L2 flushed:
python scripts/k0_time.py  (same measurement as bench.py secondary_config3)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1701_08547_b200 import batch, workloads  # noqa: E402

c = workloads.make_corpus(100_000)
rec = workloads.corpus_records(c)
lut = workloads.corpus_signature_lut()
byts = 4 * c.n_instr + 8 * (c.n_kernels + 1) + 144 * c.n_kernels
peak = json.load(open(os.path.join(os.path.dirname(bench.__file__), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6547.5
for name, r, l in (("class", batch.classify_records(rec, lut), batch.CLASS_LUT), ("sig", rec, lut)):
    ms = [bench._k0_time(c, r, l, reps=20) for _ in range(3)]
    print(f"K0 {name}: ms {['%.4f' % m for m in ms]} frac {byts / (min(ms) / 1e3) / 1e9 / peak:.3f}")
