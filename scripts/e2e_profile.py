"""Host-side breakdown of one score_space() step (config 5): the native pack
(_SpacePack), the one-call occx_score_space_host (H2D, K1, feature table,
K2i, K3, D2H, wait) and the native decode.

    python scripts/e2e_profile.py [--every-key]
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1701_08547_b200 import score_space, workloads  # noqa: E402
from paper_1701_08547_b200.batch import _SpacePack, space_score  # noqa: E402

PRUNE = "--every-key" not in sys.argv
cfg = workloads.config5()
for _ in range(5):
    score_space(cfg.kernels, cfg.archs, prune=PRUNE)
torch.cuda.synchronize()
rows = []
for _ in range(30):
    t0 = time.perf_counter()
    pk = _SpacePack(cfg.kernels, cfg.archs, 16)
    t1 = time.perf_counter()
    segs, keys = space_score(pk, prune=PRUNE, to_host=True)
    t2 = time.perf_counter()
    rows.append((t1 - t0, t2 - t1, t2 - t0))
tot = []
for _ in range(30):
    t0 = time.perf_counter()
    score_space(cfg.kernels, cfg.archs, prune=PRUNE)
    tot.append(time.perf_counter() - t0)
dec = []
for _ in range(30):
    t0 = time.perf_counter()
    pk.decode(keys)
    dec.append(time.perf_counter() - t0)
med = [statistics.median(r[i] for r in rows) * 1e3 for i in range(3)]
print(f"prune={PRUNE}: pack {med[0]:.3f} ms | score_space_host + decode {med[1]:.3f} | "
      f"decode alone {statistics.median(dec) * 1e3:.3f} | score_space() total "
      f"{statistics.median(tot) * 1e3:.3f} ms")
