"""K2 time per segment of config 5 (64,225,280 candidates each, back-to-back
launches), to see which (kernel, arch) content is compute-heavy.

    python scripts/k2_segments.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1701_08547_b200 import ScorePlan, workloads  # noqa: E402

cfg = workloads.config5()
plan = ScorePlan(cfg.kernels, cfg.archs, k=cfg.k)
rec = plan.generate()
torch.cuda.synchronize()
seg = plan.total // plan.n_seg
for s in range(plan.n_seg):
    b = s * seg
    view = rec[16 * b:]
    for _ in range(2):
        plan.score_partials(view, seg, index_base=b)
    torch.cuda._sleep(1_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        plan.score_partials(view, seg, index_base=b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    k, a = divmod(s, plan.n_arch)
    print(f"seg {s:2d} {cfg.kernels[k].name:9s} {cfg.archs[a].name:12s} {ms:.4f} ms "
          f"{16 * seg / ms / 1e6:7.0f} GB/s", flush=True)
