"""Three K2 launches on rank g's shard of config 5 at G ranks (an ncu
target: ncu -k regex:score_topk_tma -s 2 -c 1 python scripts/k2_one_shard.py g G)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1701_08547_b200 import ScorePlan, workloads  # noqa: E402
from paper_1701_08547_b200.dist import shard_range  # noqa: E402

g, G = int(sys.argv[1]), int(sys.argv[2])
cfg = workloads.config5()
plan = ScorePlan(cfg.kernels, cfg.archs, k=cfg.k)
b, e = shard_range(plan.total, g, G)
rec = plan.generate(b, e - b)
for _ in range(3):
    plan.score_partials(rec, e - b, index_base=b)
torch.cuda.synchronize()
