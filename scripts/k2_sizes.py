"""K2 time vs call size (prefixes of config 5): back-to-back launches between
one event pair (no host gaps), and single launches behind a busy kernel.
Separates the per-call fixed cost from the streaming rate.

    python scripts/k2_sizes.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1701_08547_b200 import ScorePlan, workloads  # noqa: E402

cfg = workloads.config5()
opts = int(os.environ.get("K2_OPTIONS", "0"), 0)
plan = ScorePlan(cfg.kernels, cfg.archs, k=cfg.k, options=opts)
rec = plan.generate()
torch.cuda.synchronize()
for n in (4096, 1 << 20, 1 << 24, 1 << 26, 160_563_200, 321_126_400, 642_252_800, plan.total):
    for _ in range(3):
        plan.score_partials(rec, n)
    reps = 20 if n < (1 << 28) else 5
    torch.cuda._sleep(1_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.score_partials(rec, n)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"n={n:>11d} ({16 * n / 1e9:7.3f} GB): K2 back-to-back {ms * 1e3:9.1f} us "
          f"-> {16 * n / ms / 1e6 if ms else 0:8.1f} GB/s", flush=True)
