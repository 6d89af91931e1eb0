import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import torch
from paper_1701_08547_b200 import score_space, workloads, ScorePlan
cfg = workloads.config5()
for _ in range(3):
    score_space(cfg.kernels, cfg.archs)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    score_space(cfg.kernels, cfg.archs)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(35)
t0 = time.perf_counter()
for _ in range(5):
    plan = ScorePlan(cfg.kernels, cfg.archs)
torch.cuda.synchronize()
print("ScorePlan ms", (time.perf_counter() - t0) / 5 * 1e3)
keys = plan.score_implicit()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    plan.decode(keys)
print("decode ms", (time.perf_counter() - t0) / 5 * 1e3)
