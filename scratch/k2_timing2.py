"""Does the K2 CTA imbalance follow the data or the SM?  config 2 scored
(a) as is, (b) with records rotated by half a CTA chunk, (c) with every
record equal to record 0 (no data dependence).  OCCX_LIB = timing build."""
import ctypes
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1701_08547_b200 import ScorePlan, _lib, workloads

lib = _lib.load()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
name = sys.argv[1] if len(sys.argv) > 1 else "config2"
cfg = workloads.CONFIGS[name]()
plan = ScorePlan(cfg.kernels, cfg.archs, "corrected", k=cfg.k)
rec = plan.generate()
n = plan.total
tiles = -(-n // 2048)
chunk = -(-tiles // 148) * 2048
v = rec.view(-1, 16)
variants = {"as-is": rec,
            "rot-half": torch.roll(v, shifts=chunk // 2, dims=0).reshape(-1).contiguous(),
            "rot-3chunks": torch.roll(v, shifts=3 * chunk, dims=0).reshape(-1).contiguous(),
            "constant": v[:1].expand(n, 16).reshape(-1).contiguous()}
for tag, r in variants.items():
    ms = []
    for rep in range(5):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.score_partials(r, n)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    buf = np.zeros(4 * 1024, np.uint64)
    lib.occx_debug_k2_timing(ctypes.c_void_p(buf.ctypes.data), 1024)
    t = buf.reshape(-1, 4)[:148].astype(np.int64)
    dur = (t[:, 1] - t[:, 0]) / 1e3
    print(f"== {name} {tag}: {np.median(ms):.4f} ms; dur min/med/max {dur.min():.0f}/{np.median(dur):.0f}/{dur.max():.0f} us")
    print("   blk:dur " + " ".join(f"{i}:{d:.0f}" for i, d in enumerate(dur)))
    print("   sm of slowest 10:", [int(t[i, 2]) for i in np.argsort(dur)[-10:]], flush=True)
