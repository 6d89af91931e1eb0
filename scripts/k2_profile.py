"""K2 (record scorer) timing by call size, and -- with the instrumented build
(`python -m paper_1701_08547_b200.build --timing`, loaded through
OCCX_LIB=paper_1701_08547_b200/_objs_timing/liboccx_timing.so) -- the
per-CTA globaltimer spans and slow-path counters.

    python scripts/k2_profile.py [workload ...]

workloads: config2, config4, config5, shard8 (the first 1/8 of config 5,
one rank's strong-scaling shard at G = 8).  Prints per workload: K2 alone,
K2 + K3, per-candidate ps, and (timing build) CTA start/end spread.
"""

import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_08547_b200 import ScorePlan, _lib, workloads  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
lib = _lib.load()
timing = hasattr(lib, "occx_debug_k2_timing") and "timing" in (os.environ.get("OCCX_LIB") or "")


def timed(fn, reps=15, do_flush=True):
    """GPU time of one launch.  The start event is queued behind a busy
    kernel (the L2 flush, or a 200 us spin when the input is far above L2),
    so the host's launch overhead is not inside the events."""
    ts = []
    for _ in range(reps):
        if do_flush:
            flush.fill_(1)
        else:
            torch.cuda._sleep(400_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def workload(name):
    if name.startswith("seg"):               # one segment of config 5: seg<s>
        cfg = workloads.config5()
        size = cfg.total // 20
        return cfg, int(name[3:]) * size, size
    if name == "shard8":
        cfg = workloads.config5()
        total = cfg.total
        return cfg, 0, -(-total // 8)
    cfg = workloads.CONFIGS[name]()
    return cfg, 0, None


def main():
    names = sys.argv[1:] or ["config2", "config4", "shard8", "config5"]
    for name in names:
        cfg, begin, n = workload(name)
        plan = ScorePlan(cfg.kernels, cfg.archs, "corrected", k=cfg.k,
                         options=int(os.environ.get("K2_OPTIONS", "0"), 0))
        n = plan.total if n is None else n
        rec = plan.generate(begin, n)
        out = torch.empty((plan.n_seg, plan.k), dtype=torch.int64, device="cuda")
        for _ in range(3):
            plan.score(rec, n, index_base=begin, out=out)
        torch.cuda.synchronize()
        big = 16 * n > (1 << 30)
        k2 = timed(lambda: plan.score_partials(rec, n, index_base=begin), do_flush=not big)
        k23 = timed(lambda: plan.score(rec, n, index_base=begin, out=out), do_flush=not big)
        gb = 16 * n / 1e9
        print(f"{name}: n={n} K2 {k2:.4f} ms ({gb / k2 * 1e3:.0f} GB/s, {k2 * 1e9 / n:.3f} ps/cand)"
              f"  K2+K3 {k23:.4f} ms  ideal@7150GB/s {gb / 7150 * 1e3:.4f} ms", flush=True)
        if timing:
            plan.score_partials(rec, n, index_base=begin)
            torch.cuda.synchronize()
            buf = np.zeros(8 * 1024, np.uint64)
            lib.occx_debug_k2_timing(ctypes.c_void_p(buf.ctypes.data), 1024)
            t = buf.reshape(-1, 8)[: plan.grid_lists].astype(np.int64)
            t0 = t[:, 0].min()
            ent, setup, cons, end = [(t[:, i] - t0) / 1e3 for i in range(4)]

            def mmm(x):
                return f"{x.min():.1f}/{np.median(x):.1f}/{x.max():.1f}"
            print(f"   us since first CTA entry (min/med/max): entry {mmm(ent)}; setup done "
                  f"{mmm(setup)}; consumers done {mmm(cons)}; end {mmm(end)}")
            print(f"   per CTA: setup {mmm(setup - ent)}; stream {mmm(cons - setup)}; "
                  f"merge+flush {mmm(end - cons)}")
            cnt = np.zeros(8 * 1024, np.uint64)
            plan.score_partials(rec, n, index_base=begin)
            torch.cuda.synchronize()
            lib.occx_debug_k2_counts(ctypes.c_void_p(cnt.ctypes.data), 1024, 1)
            plan.score_partials(rec, n, index_base=begin)
            torch.cuda.synchronize()
            lib.occx_debug_k2_counts(ctypes.c_void_p(cnt.ctypes.data), 1024, 1)
            c = cnt.reshape(-1, 8)[: plan.grid_lists].sum(axis=0)
            print(f"   per launch: offers {c[0]} (per 1M cand {c[0] / n * 1e6:.0f}), batch merges "
                  f"{c[1]}, segment flushes {c[2]}, mixed batches {c[3]}, CTA inserts {c[4]}, "
                  f"cache fills {c[5]} ({c[5] / n * 1e6:.0f}/M), offer cycles {c[6] / max(c[0], 1):.0f}"
                  f"/offer, full-wait cycles/warp {c[7] / plan.grid_lists / 16:.0f}")
            dur = cons - setup
            slow = np.argsort(dur)[-8:]
            print("   slowest streams (blk:us:tiles):",
                  " ".join(f"{i}:{dur[i]:.0f}:{t[i, 5]}" for i in slow), flush=True)


if __name__ == "__main__":
    main()
