"""K2 time of each rank's shard of config 5 at G = 2, 4, 8 (strong scaling:
contiguous index ranges, records decoded into HBM), back-to-back launches.
The slowest shard sets the G-GPU step.

    python scripts/k2_shards.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1701_08547_b200 import ScorePlan, workloads  # noqa: E402
from paper_1701_08547_b200.dist import shard_range  # noqa: E402

cfg = workloads.config5()
plan = ScorePlan(cfg.kernels, cfg.archs, k=cfg.k,
                 options=int(os.environ.get("K2_OPTIONS", "0"), 0))
rec = plan.generate()
torch.cuda.synchronize()


def k2_ms(begin, n, reps=10):
    view = rec[16 * begin:]
    for _ in range(2):
        plan.score_partials(view, n, index_base=begin)
    torch.cuda._sleep(1_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.score_partials(view, n, index_base=begin)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


full = k2_ms(0, plan.total, 5)
print(f"G=1: {full:.4f} ms ({plan.total * 1e-9 / full * 1e3 * 1e-3:.1f} G/ms)")
for G in (2, 4, 8):
    ts = []
    for g in range(G):
        b, e = shard_range(plan.total, g, G)
        ts.append(k2_ms(b, e - b))
    print(f"G={G}: shards " + " ".join(f"{t:.4f}" for t in ts) +
          f"  max {max(ts):.4f} ms -> K2-only strong-scaling efficiency "
          f"{full / G / max(ts) * 100:.1f} %", flush=True)
