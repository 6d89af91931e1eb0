"""Where the host time of score_space_multi goes (config 5, N=1)."""
import cProfile
import pstats
import sys
import time
sys.path.insert(0, '.')
import torch
from paper_1701_08547_b200 import workloads
from paper_1701_08547_b200.batch import ScorePlan
from paper_1701_08547_b200.dist import score_space_multi

cfg = workloads.config5()
for _ in range(3):
    score_space_multi(cfg.kernels, cfg.archs, "corrected", cfg.k, scaling="weak")
torch.cuda.synchronize()
N = 20
acc = dict(plan=0.0, launch=0.0, tables=0.0, d2h=0.0, decode=0.0)
for _ in range(N):
    t0 = time.perf_counter()
    p = ScorePlan(cfg.kernels, cfg.archs, "corrected", cfg.k)
    t1 = time.perf_counter()
    keys = p.score_implicit(0, p.total, key_offset=0)
    t2 = time.perf_counter()
    p.decode_tables()
    t3 = time.perf_counter()
    kh = keys.cpu()
    t4 = time.perf_counter()
    p.decode(kh)
    t5 = time.perf_counter()
    for k_, v in zip(acc, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)):
        acc[k_] += v
print({k_: round(v / N * 1e3, 3) for k_, v in acc.items()}, "ms")
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    score_space_multi(cfg.kernels, cfg.archs, "corrected", cfg.k, scaling="weak")
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
