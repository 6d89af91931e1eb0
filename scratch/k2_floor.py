"""K2's memory floor on config 5: the same kernel over records that are all
equal (no data-dependent work) vs the real records, and a plain
device-to-device copy of the same bytes for the read+write reference."""
import sys
sys.path.insert(0, '.')
import statistics
import torch
from paper_1701_08547_b200 import ScorePlan, workloads

cfg = workloads.config5()
plan = ScorePlan(cfg.kernels, cfg.archs, "corrected", k=cfg.k)
rec = plan.generate()
n = plan.total


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


real = timed(lambda: plan.score_partials(rec, n))
const = rec.view(-1, 16)[:1].expand(n, 16).reshape(-1).contiguous()
flat = timed(lambda: plan.score_partials(const, n))
del const
dst = torch.empty_like(rec)
cp = timed(lambda: dst.copy_(rec))
gb = 16 * n / 1e9
print(f"K2 real {real:.3f} ms ({gb / real * 1e3:.0f} GB/s)  K2 constant records {flat:.3f} ms ({gb / flat * 1e3:.0f} GB/s)  "
      f"D2D copy {cp:.3f} ms ({2 * gb / cp * 1e3:.0f} GB/s read+write)")
