"""Rank g's shard of config 5 (G = 8) scored from its own 2.57 GB allocation
(what a rank of the multi-GPU bench does) vs as a view into the full 20.5 GB
array (scripts/k2_shards.py), plus the stream-only build for reference.

    python scripts/k2_shard_alloc.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1701_08547_b200 import ScorePlan, workloads  # noqa: E402
from paper_1701_08547_b200.dist import shard_range  # noqa: E402

cfg = workloads.config5()
plan = ScorePlan(cfg.kernels, cfg.archs, k=cfg.k)


def t(rec, b, n, reps=10):
    for _ in range(3):
        plan.score_partials(rec, n, index_base=b)
    torch.cuda._sleep(1_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.score_partials(rec, n, index_base=b)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for g in (0, 1):
    b, e = shard_range(plan.total, g, 8)
    own = plan.generate(b, e - b)
    torch.cuda.synchronize()
    print(f"shard {g}: own allocation {t(own, b, e - b):.4f} ms", flush=True)
    del own
full = plan.generate()
for g in (0, 1):
    b, e = shard_range(plan.total, g, 8)
    print(f"shard {g}: view of the full array {t(full[16 * b:], b, e - b):.4f} ms", flush=True)
print(f"full: {t(full, 0, plan.total, 5):.4f} ms")
