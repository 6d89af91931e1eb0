"""Per-CTA slow-path counters of K2 (timing build): which path makes the
CTAs holding a segment boundary slow?"""
import ctypes
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1701_08547_b200 import ScorePlan, _lib, workloads

lib = _lib.load()
NAMES = ["offer", "ins_iter", "adopt", "mixed", "cta_ins", "fill", "slow_clk", "wait_clk"]
for name in sys.argv[1:] or ["config2"]:
    cfg = workloads.CONFIGS[name]()
    plan = ScorePlan(cfg.kernels, cfg.archs, "corrected", k=cfg.k)
    rec = plan.generate()
    cnt = np.zeros(8 * 1024, np.uint64)
    lib.occx_debug_k2_counts(ctypes.c_void_p(cnt.ctypes.data), 1024, 1)
    plan.score_partials(rec, plan.total)
    torch.cuda.synchronize()
    hist = np.zeros(16 * 1024, np.uint64)
    lib.occx_debug_k2_hist(ctypes.c_void_p(hist.ctypes.data), 1024)
    lib.occx_debug_k2_counts(ctypes.c_void_p(cnt.ctypes.data), 1024, 1)
    buf = np.zeros(4 * 1024, np.uint64)
    lib.occx_debug_k2_timing(ctypes.c_void_p(buf.ctypes.data), 1024)
    t = buf.reshape(-1, 4)[:148].astype(np.int64)
    dur = (t[:, 1] - t[:, 0]) / 1e3
    c = cnt.reshape(-1, 8)[:148, :8].astype(np.int64)
    print(f"== {name}: totals " + ", ".join(f"{n}={int(c[:, i].sum())}" for i, n in enumerate(NAMES)))
    for b in list(np.argsort(dur)[:4]) + list(np.argsort(dur)[-6:]):
        print(f"  blk {b:3d} {dur[b]:7.1f} us  " + " ".join(f"{n}={int(c[b, i])}" for i, n in enumerate(NAMES)))
    sys.stdout.flush()
    hh = hist.reshape(-1, 16)[:148].astype(np.int64)
    chunk = -(-(-(-plan.total // 2048)) // 148) * 2048
    seg_len = plan.total // plan.n_seg
    for b in list(np.argsort(dur)[:2]) + list(np.argsort(dur)[-3:]):
        lo = b * chunk
        bpos = ((lo // seg_len + 1) * seg_len - lo) / chunk
        print(f"  blk {b:3d} boundary at {bpos:.2f} of chunk; process kcycles/bucket:",
              " ".join(str(int(x) // 1000) for x in hh[b]))
