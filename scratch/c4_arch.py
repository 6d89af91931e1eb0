import sys
sys.path.insert(0, '.')
import torch
from paper_1701_08547_b200 import ScorePlan, workloads
cfg = workloads.config4()
for ai, a in enumerate(cfg.archs):
    plan = ScorePlan(cfg.kernels, [a], k=16)
    rec = plan.generate()
    for _ in range(3): plan.score(rec, plan.total)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): plan.score_partials(rec, plan.total)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"arch {a.name}: {plan.total} cand, K2 {ms:.3f} ms, {plan.total/ms/1e6:.1f} G/s, {16*plan.total/ms/1e6:.0f} GB/s")
for ki, k in enumerate(cfg.kernels):
    plan = ScorePlan([k], cfg.archs, k=16)
    rec = plan.generate()
    for _ in range(3): plan.score(rec, plan.total)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): plan.score_partials(rec, plan.total)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"kernel {k.name}: K2 {ms:.3f} ms, {plan.total/ms/1e6:.1f} G/s")
