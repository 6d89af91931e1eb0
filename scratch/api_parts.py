import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1701_08547_b200 import workloads, batch
from paper_1701_08547_b200.batch import ScorePlan
cfg = workloads.config5()
for _ in range(3):
    p = ScorePlan(cfg.kernels, cfg.archs); p.decode(p.score_implicit())
torch.cuda.synchronize()
import paper_1701_08547_b200.batch as B
# monkeypatch timers into ScorePlan pieces
T = {}
def tic(): return time.perf_counter()
N = 20
acc = {"plan": 0, "launch": 0, "wait": 0, "decode": 0}
for _ in range(N):
    t0 = tic(); p = ScorePlan(cfg.kernels, cfg.archs); t1 = tic()
    keys = p.score_implicit(); t2 = tic()
    kh = keys.cpu(); t3 = tic()
    p.decode(kh); t4 = tic()
    acc["plan"] += t1 - t0; acc["launch"] += t2 - t1; acc["wait"] += t3 - t2; acc["decode"] += t4 - t3
print({k: round(v / N * 1e3, 3) for k, v in acc.items()})
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(20): ScorePlan(cfg.kernels, cfg.archs)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
