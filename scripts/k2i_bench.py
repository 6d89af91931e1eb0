import sys, time, torch
sys.path.insert(0, '.')
from paper_1701_08547_b200 import ScorePlan, workloads
for name in ("config4", "config5"):
    cfg = workloads.CONFIGS[name]()
    plan = ScorePlan(cfg.kernels, cfg.archs, k=16)
    for _ in range(3): plan.score_implicit()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): plan.score_implicit()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{name} K2i {ms:.3f} ms  {plan.total/ms/1e6:.1f} G cand/s")
    t0 = time.perf_counter()
    for _ in range(5):
        from paper_1701_08547_b200 import score_space
        res = score_space(cfg.kernels, cfg.archs)
    dt = (time.perf_counter() - t0) / 5
    print(f"{name} score_space() end-to-end {dt*1e3:.1f} ms  {plan.total/dt/1e9:.1f} G cand/s")
