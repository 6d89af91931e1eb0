"""K2 + K3 (ScorePlan.score) on config 5: full size and the G = 8 shards
(strong scaling, contiguous index ranges), back-to-back launches.
    python scripts/k2k3_time.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_08547_b200 import ScorePlan, workloads  # noqa: E402
from paper_1701_08547_b200.dist import shard_range  # noqa: E402

cfg = workloads.config5()
plan = ScorePlan(cfg.kernels, cfg.archs, k=cfg.k)
rec = plan.generate()
torch.cuda.synchronize()


def ms(b, n, reps=10):
    view = rec[16 * b:]
    for _ in range(3):
        plan.score(view, n, index_base=b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.score(view, n, index_base=b)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


full = ms(0, plan.total, 10)
ts = [ms(*(lambda r: (r[0], r[1] - r[0]))(shard_range(plan.total, g, 8))) for g in range(8)]
print(f"full {full:.4f} ms; G8 shards " + " ".join(f"{t:.4f}" for t in ts) +
      f"; slowest rate vs full {full / 8 / max(ts):.3f}")
