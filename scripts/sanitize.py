"""Workload for compute-sanitizer (racecheck / synccheck / memcheck / initcheck):
one small call of every liboccx kernel, each result checked against the
oracle or the record path, so a hazard report comes with a correct run.

    compute-sanitizer --tool racecheck --racecheck-report all \
        --kernel-name regex='score_|topk_merge|mix_reduce|feature_kernel|occ_dump|suggest_kernel|build_vtab|gen_space' \
        python scripts/sanitize.py

Covers K0 (mix_reduce), K1 (feature_kernel), vtab build, K2 with the TMA
ring (two slices and one slice) and with the LDG feed, K2i with block
pruning on and off, K3 (topk_merge), Kd, K4 and the generator, on config 1,
a window of config 2 (segment boundaries inside CTA chunks) and a random
arch table (tests/test_gpu_random.py's generator).
"""

import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1701_08547_b200 import ScorePlan, _lib, batch, workloads  # noqa: E402


def check_plan(cfg, begin, n, name):
    want = None
    for options in (0, _lib.CTX_K2_ONE_SLICE, _lib.CTX_K2_FEED_LDG):
        plan = ScorePlan(cfg.kernels, cfg.archs, k=cfg.k, options=options)
        rec = plan.generate(begin, n)
        got = plan.score(rec, n, index_base=begin).cpu().numpy()
        if want is None:
            prob = oracle.problem_of(cfg)
            want = oracle.score_records(prob, rec[: n * 16].cpu().numpy(),
                                        index_base=begin).view(np.int64)
        assert np.array_equal(got, want), (name, "K2", options)
        for prune in (True, False):
            imp = plan.score_implicit(begin, n, prune=prune).cpu().numpy()
            assert np.array_equal(imp, want), (name, "K2i", prune)
    print(f"{name}: K2 (TMA 2-slice, 1-slice, LDG) + K2i (pruned, every key) + K3 ok", flush=True)


def main():
    torch.cuda.set_device(0)
    check_plan(workloads.config1(), 0, 32, "config1")
    c2 = workloads.config2()
    check_plan(c2, 1_000_003, 2_500_017, "config2 window")
    from test_gpu_random import random_config
    rc = random_config(random.Random(1003), n_arch=3, n_kern=3)
    plan = ScorePlan(rc.kernels, rc.archs, k=rc.k)
    check_plan(rc, 0, min(plan.total, 3_000_000), "random archs")

    # K0 on a corpus slice vs the C oracle
    c = workloads.make_corpus(3000)
    rec = workloads.corpus_records(c)
    lut = workloads.corpus_signature_lut()
    d_rec, d_off, d_lut = batch._to_device(rec), batch._to_device(c.offsets), batch._to_device(lut)
    out = batch._empty(c.n_kernels * _lib.MIX.itemsize)
    batch.mix_reduce(d_rec, d_off, c.n_kernels, d_lut, len(lut), d_out=out)
    got = batch._to_host(out, _lib.MIX, c.n_kernels)
    counts, _, regs = oracle.aggregate_records(rec, c.offsets, lut)
    assert np.array_equal(got["counts"][:, :15].astype(np.int64), counts), "K0 counts"
    assert np.array_equal(got["reg_operands"].astype(np.int64), regs), "K0 reg_operands"
    # class records (identity table: the byte-indexed increment path) and a
    # permuted 15-entry table (same kernel instance, generic lookups)
    crec = batch.classify_records(rec, lut)
    for tab in (batch.CLASS_LUT, np.random.default_rng(5).permutation(15).astype(np.uint8)):
        batch.mix_reduce(batch._to_device(crec), d_off, c.n_kernels, batch._to_device(tab),
                         len(tab), d_out=out)
        got = batch._to_host(out, _lib.MIX, c.n_kernels)
        counts, _, regs = oracle.aggregate_records(crec, c.offsets, tab)
        assert np.array_equal(got["counts"][:, :15].astype(np.int64), counts), "K0 class counts"
    print("K0 ok", flush=True)

    # Kd + K4
    archs = workloads.all_archs()
    ob = batch.occupancy_batch(archs[1], [(t, r, s) for t in (1, 128, 1024, 1056)
                                          for r in (0, 27, 256) for s in (0, 49153)])
    assert len(ob) == 24
    from paper_1701_08547_b200 import KernelResources
    sb = batch.suggest_batch([(a, KernelResources("k", 32, 1024)) for a in archs])
    assert len(sb) == len(archs)
    torch.cuda.synchronize()
    print("Kd, K4 ok; sanitize workload done", flush=True)


if __name__ == "__main__":
    main()
