import sys, time
sys.path.insert(0, '.')
import torch
from paper_1701_08547_b200 import workloads, batch
cfg = workloads.config5()
for _ in range(5): batch.ScorePlan(cfg.kernels, cfg.archs)
torch.cuda.synchronize(); batch.PLAN_T.clear()
for _ in range(50): batch.ScorePlan(cfg.kernels, cfg.archs)
print({k: round(v / 50 * 1e3, 3) for k, v in batch.PLAN_T.items()})
