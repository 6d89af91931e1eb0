"""Where a scalar occupancy() call spends its time (GPU box):
python scripts/scalar_breakdown.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_08547_b200 import LaunchInput, _lib, batch, occupancy, workloads  # noqa: E402
from paper_1701_08547_b200.batch import MODE_CODE, Mode  # noqa: E402

arch = workloads.all_archs()[1]
li = LaunchInput(256, 32, 4096)
lib = _lib.load()


def t(fn, n=3000):
    for _ in range(200):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


_, page, base = batch._lane()
h_archs = batch._packed_archs((arch,))
ctx, sp = _lib.ctx(), _lib.stream_ptr()


def raw():
    lib.occx_occupancy_batch(ctx, h_archs.ctypes.data, 1, base, 1, 0, base + 256, sp)
    lib.occx_stream_sync(sp)


def launch_only():
    lib.occx_occupancy_batch(ctx, h_archs.ctypes.data, 1, base, 1, 0, base + 256, sp)


x = torch.zeros(1, device="cuda")
print(f"occupancy() {t(lambda: occupancy(arch, li)):.1f} us")
print(f"occupancy_single() {t(lambda: batch.occupancy_single(arch, 256, 32, 4096)):.1f} us")
print(f"ctypes launch + sync {t(raw):.1f} us")
print(f"ctypes launch only {t(launch_only):.1f} us")
torch.cuda.synchronize()
print(f"stream sync alone {t(lambda: lib.occx_stream_sync(sp)):.1f} us")
print(f"_packed_archs {t(lambda: batch._packed_archs((arch,))):.1f} us")
print(f"torch add_ + synchronize {t(lambda: (x.add_(1), torch.cuda.synchronize())):.1f} us")
