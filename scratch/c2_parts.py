"""K2 vs K3 split and per-CTA balance on configs 2 and 4 (records resident)."""
import sys
sys.path.insert(0, '.')
import statistics
import torch
from paper_1701_08547_b200 import ScorePlan, workloads

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=15, do_flush=True):
    ts = []
    for _ in range(reps):
        if do_flush:
            flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for name in sys.argv[1:] or ["config2", "config4"]:
    cfg = workloads.CONFIGS[name]()
    plan = ScorePlan(cfg.kernels, cfg.archs, "corrected", k=cfg.k)
    rec = plan.generate()
    for _ in range(3):
        plan.score(rec, plan.total)
    torch.cuda.synchronize()
    k2 = timed(lambda: plan.score_partials(rec, plan.total))
    k23 = timed(lambda: plan.score(rec, plan.total))
    k23_nf = timed(lambda: plan.score(rec, plan.total), do_flush=False)
    gb = 16 * plan.total / 1e9
    print(f"{name}: n={plan.total} K2 {k2:.4f} ms ({gb / k2 * 1e3:.0f} GB/s)  K2+K3 {k23:.4f} ms"
          f"  K2+K3 no flush {k23_nf:.4f} ms  ideal@6537 {gb / 6537 * 1e3:.4f} ms", flush=True)
