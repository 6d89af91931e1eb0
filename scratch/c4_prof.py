import sys
sys.path.insert(0, '.')
import torch
from paper_1701_08547_b200 import ScorePlan, workloads
cfg = workloads.config4()
plan = ScorePlan(cfg.kernels, cfg.archs, k=16)
rec = plan.generate()
for _ in range(5):
    plan.score(rec, plan.total)
torch.cuda.synchronize()
