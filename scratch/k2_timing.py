"""Per-CTA K2 start/end times (globaltimer) on configs 2/4: is the tail
imbalance data, placement or memory?  Needs OCCX_LIB=scratch/k2lib/liboccx_timing.so."""
import ctypes
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1701_08547_b200 import ScorePlan, _lib, workloads

lib = _lib.load()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for name in sys.argv[1:] or ["config2", "config4"]:
    cfg = workloads.CONFIGS[name]()
    plan = ScorePlan(cfg.kernels, cfg.archs, "corrected", k=cfg.k)
    rec = plan.generate()
    for rep in range(4):
        flush.fill_(1)
        torch.cuda.synchronize()
        plan.score_partials(rec, plan.total)
        torch.cuda.synchronize()
    buf = np.zeros(4 * 1024, np.uint64)
    lib.occx_debug_k2_timing(ctypes.c_void_p(buf.ctypes.data), 1024)
    t = buf.reshape(-1, 4)[:148].astype(np.int64)
    t0 = t[:, 0].min()
    st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
    dur = en - st
    print(f"== {name}: start spread {st.max():.1f} us, end min/med/max {en.min():.1f}/"
          f"{np.median(en):.1f}/{en.max():.1f} us, tiles {sorted(set(t[:, 3].tolist()))}")
    order = np.argsort(dur)
    print("  fastest CTAs (blk, sm, us):", [(int(i), int(t[i, 2]), round(float(dur[i]), 1)) for i in order[:8]])
    print("  slowest CTAs (blk, sm, us):", [(int(i), int(t[i, 2]), round(float(dur[i]), 1)) for i in order[-8:]])
    print("  duration by block id (x10):", [round(float(x), 0) for x in dur[::10]])
    sm = t[:, 2]
    print("  duration by smid parity even/odd:", round(float(dur[sm % 2 == 0].mean()), 1), round(float(dur[sm % 2 == 1].mean()), 1))
    print("  sm<74 vs >=74:", round(float(dur[sm < 74].mean()), 1), round(float(dur[sm >= 74].mean()), 1), flush=True)
