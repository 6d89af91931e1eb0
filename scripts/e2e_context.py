"""score_space() e2e time in three contexts: fresh process, after 20 K2 steps
over config 5's 20.5 GB of records (bench order), and with those records
freed again -- to explain bench's e2e vs scripts/e2e_profile.py.

    python scripts/e2e_context.py
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1701_08547_b200 import ScorePlan, score_space, workloads  # noqa: E402

cfg = workloads.config5()


def e2e(tag, n=40):
    for _ in range(5):
        score_space(cfg.kernels, cfg.archs, prune=False)
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        score_space(cfg.kernels, cfg.archs, prune=False)
        ts.append(time.perf_counter() - t0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        score_space(cfg.kernels, cfg.archs, prune=False)
    e1.record()
    torch.cuda.synchronize()
    print(f"{tag}: median {statistics.median(ts) * 1e3:.3f} ms, min {min(ts) * 1e3:.3f}, "
          f"events {e0.elapsed_time(e1) / n:.3f} ms", flush=True)


e2e("fresh")
plan = ScorePlan(cfg.kernels, cfg.archs, k=cfg.k)
rec = plan.generate()
for _ in range(25):
    plan.score(rec, plan.total)
torch.cuda.synchronize()
e2e("after 25 K2 steps, records resident")
del rec
torch.cuda.empty_cache()
e2e("records freed")
