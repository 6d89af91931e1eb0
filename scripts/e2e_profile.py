"""Host-side breakdown of one score_space() step (config 5): plan build
(pack + H2D + K1 + feature table launches), K2i + K3 launch, D2H wait,
decode; plus the same step with CUDA events around the GPU part.

    python scripts/e2e_profile.py [--every-key]
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1701_08547_b200 import ScorePlan, workloads  # noqa: E402
from paper_1701_08547_b200 import batch  # noqa: E402

PRUNE = "--every-key" not in sys.argv
cfg = workloads.config5()
for _ in range(5):
    ScorePlan(cfg.kernels, cfg.archs).decode(
        ScorePlan(cfg.kernels, cfg.archs).score_implicit(prune=PRUNE).cpu())
torch.cuda.synchronize()
rows = []
for _ in range(30):
    t0 = time.perf_counter()
    plan = ScorePlan(cfg.kernels, cfg.archs)
    t1 = time.perf_counter()
    d = plan.score_implicit(prune=PRUNE)
    t2 = time.perf_counter()
    keys = d.cpu()
    t3 = time.perf_counter()
    plan.decode(keys)
    t4 = time.perf_counter()
    rows.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0))
med = [statistics.median(r[i] for r in rows) * 1e3 for i in range(5)]
print(f"prune={PRUNE}: plan {med[0]:.3f} ms | score launch {med[1]:.3f} | D2H wait {med[2]:.3f} "
      f"| decode {med[3]:.3f} | total {med[4]:.3f} ms")
# pieces of the plan build
pk = []
for _ in range(30):
    t0 = time.perf_counter()
    batch._host().pack_plan(
        [(k.space.thread_counts, k.space.block_counts, k.space.unroll_factors,
          k.space.l1_sizes_kb, k.space.compiler_flags, dict(k.space.extra)["REGS"],
          dict(k.space.extra)["SMEM"]) for k in cfg.kernels],
        [len(k.mixes) for k in cfg.kernels], [m for k in cfg.kernels for m in k.mixes],
        [batch.thread_candidates(a) for a in cfg.archs], batch.DEVICE_ID, batch.DeviceError)
    pk.append(time.perf_counter() - t0)
print(f"pack_plan alone {statistics.median(pk) * 1e3:.3f} ms")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        plan = ScorePlan(cfg.kernels, cfg.archs)
        plan.decode(plan.score_implicit(prune=PRUNE).cpu())
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=20))
