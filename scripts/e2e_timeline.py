"""GPU timeline of score_space() steps (config 5) from CUPTI via
torch.profiler: kernels and copies with start offsets and durations, so the
gaps between them (launch latency, host work) are visible.
    python scripts/e2e_timeline.py [--every-key]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1701_08547_b200 import score_space, workloads  # noqa: E402

PRUNE = "--every-key" not in sys.argv
cfg = workloads.config5()
for _ in range(5):
    score_space(cfg.kernels, cfg.archs, prune=PRUNE)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        score_space(cfg.kernels, cfg.archs, prune=PRUNE)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev = None
for e in evs:
    s, d = e.time_range.start - t0, e.time_range.elapsed_us()
    gap = s - prev if prev is not None else 0
    print(f"{s:9.1f} us  gap {gap:7.1f}  dur {d:8.1f}  {e.name[:70]}")
    prev = s + d
