"""K2i timing (config 4, 5) and score_space() end to end.
    python scripts/k2i_bench.py [--every-key]   (--every-key: no block pruning)"""
import sys, time, torch
sys.path.insert(0, '.')
PRUNE = "--every-key" not in sys.argv
from paper_1701_08547_b200 import ScorePlan, workloads
for name in ("config4", "config5"):
    cfg = workloads.CONFIGS[name]()
    plan = ScorePlan(cfg.kernels, cfg.archs, k=16)
    for _ in range(3): plan.score_implicit(prune=PRUNE)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): plan.score_implicit(prune=PRUNE)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{name} K2i {ms:.3f} ms  {plan.total/ms/1e6:.1f} G cand/s")
    t0 = time.perf_counter()
    for _ in range(5):
        from paper_1701_08547_b200 import score_space
        res = score_space(cfg.kernels, cfg.archs, prune=PRUNE)
    dt = (time.perf_counter() - t0) / 5
    print(f"{name} score_space() end-to-end {dt*1e3:.1f} ms  {plan.total/dt/1e9:.1f} G cand/s")
