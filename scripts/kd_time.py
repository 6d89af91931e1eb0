"""Kd over the acceptance-7a sweep (records resident, L2 flushed), as in
bench.py secondary_acceptance_7a: python scripts/kd_time.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1701_08547_b200 import _lib, batch  # noqa: E402

archs, launches, arch_index = bench._sweep_7a()
n = len(launches)
d_rec = batch._to_device(batch.pack_launches(launches, arch_index))
out = batch._empty(n * _lib.OCC.itemsize)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    batch.occupancy_records(archs, d_rec, n, d_out=out)
for _ in range(3):
    ts = []
    for _ in range(20):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        batch.occupancy_records(archs, d_rec, n, d_out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    print(f"Kd {ms * 1e3:.1f} us, frac {n * 48 / (ms / 1e3) / 1e9 / 6548.8:.3f}")
