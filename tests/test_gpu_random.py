"""Randomised GPU parity: random architecture tables (anything the packed
device form can represent), random tuning spaces, random instruction mixes,
both evaluation modes -- CUDA path vs the independent oracles.  Seeded, so
a failure reproduces."""

import os
import random

import numpy as np
import pytest

import oracle
from oracle import pyref

pytestmark = pytest.mark.gpu


def random_arch(rng, i):
    from paper_1701_08547_b200.arch import ArchSpec, Family
    ws = rng.choice((8, 16, 32, 32, 32, 64))
    wpb_max = rng.randint(1, min(64, 2048 // ws))          # device tables: T <= 2048
    tmax = ws * wpb_max
    wmp = rng.randint(1, min(127, max(1, 4096 // ws)))
    bmp = rng.randint(1, 255)
    rfs = rng.choice((16384, 32768, 65536, 131072, rng.randint(1024, (1 << 20) - 1)))
    gran = rng.choice((1, 2, 64, 128, 256, 512, rng.randint(1, 4096)))
    rmax = rng.randint(1, min(1023, rfs))
    smax = rng.choice((16384, 49152, 98304, 232448, rng.randint(1, (1 << 24) - 1)))
    cc = rng.choice((2.0, 3.5, 3.7, 5.2, 6.0, 6.1, 7.0, 9.0, 10.0))
    return ArchSpec(name=f"rand{i}", family=Family.OTHER, compute_capability=cc,
                    multiprocessors=1, warp_size=ws, max_threads_per_mp=wmp * ws,
                    max_threads_per_block=tmax, max_blocks_per_mp=bmp, max_warps_per_mp=wmp,
                    register_file_size=rfs, register_alloc_granularity=gran,
                    max_regs_per_thread=rmax, shared_mem_per_block=smax)


def random_mix(rng):
    from paper_1701_08547_b200.mix import COUNTABLE, InstructionMix
    classes = list(COUNTABLE)
    rng.shuffle(classes)
    counts = {c: rng.randint(0, 400) for c in classes[:rng.randint(0, 10)]}
    return InstructionMix(counts, rng.randint(0, 3000))


def random_config(rng, n_arch=3, n_kern=3):
    from paper_1701_08547_b200 import workloads
    from paper_1701_08547_b200.batch import KernelSpec
    from paper_1701_08547_b200.tuning import TuningSpace
    archs = tuple(random_arch(rng, i) for i in range(n_arch))
    kernels = []
    for kk in range(n_kern):
        tc = tuple(sorted(rng.sample(range(32, 2049, 32), rng.randint(1, 12))))   # masks: T <= 2048
        if rng.random() < 0.3:
            tc = tuple(rng.sample(tc, len(tc)))                  # unsorted thread dimension
        space = TuningSpace(tc, tuple(rng.sample(range(1, 300), rng.randint(1, 3))),
                            tuple(range(1, rng.randint(2, 4))), (16, 48)[:rng.randint(1, 2)],
                            ("", "-use_fast_math")[:rng.randint(1, 2)],
                            extra=(("REGS", tuple(rng.sample(range(0, 1100), rng.randint(1, 9)))),
                                   ("SMEM", tuple(rng.choice((0, 1, 1024, 6145, 49152, 232448,
                                                              rng.randint(0, 1 << 25)))
                                                  for _ in range(rng.randint(1, 6))))))
        n_var = len(space.unroll_factors) * len(space.compiler_flags)
        kernels.append(KernelSpec(f"k{kk}", space, tuple(random_mix(rng) for _ in range(n_var))))
    return workloads.Config("random", tuple(kernels), archs, rng.choice((1, 3, 16, 32)))


@pytest.mark.parametrize("seed", range(12))
def test_random_spaces_k2_k2i_vs_oracle(seed):
    import paper_1701_08547_b200 as P
    rng = random.Random(1000 + seed)
    cfg = random_config(rng, n_arch=rng.randint(1, 4), n_kern=rng.randint(1, 4))
    for mode in ("corrected", "verbatim"):
        prob = oracle.problem_of(cfg, verbatim=mode == "verbatim")
        want = oracle.score_spaces(prob, oracle.spaces_of(cfg), threads=4)
        plan = P.ScorePlan(cfg.kernels, cfg.archs, mode, k=cfg.k)
        rec = plan.generate()
        got = plan.score(rec, plan.total).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want), (seed, mode)
        for prune in (True, False):        # block-bound pruning on (default) and off
            got_i = plan.score_implicit(prune=prune).cpu().numpy().view(np.uint64)
            assert np.array_equal(got_i, want), (seed, mode, "implicit", prune)


@pytest.mark.parametrize("seed", range(6))
def test_random_archs_occupancy_vs_oracle(seed):
    from paper_1701_08547_b200.batch import occupancy_batch
    rng = random.Random(7 + seed)
    archs = [random_arch(rng, i) for i in range(8)]
    n = 200_000
    T = np.array([rng.randint(0, 2200) for _ in range(n)])
    R = np.array([rng.choice((0, rng.randint(0, 1100), rng.randint(0, 70000))) for _ in range(n)])
    S = np.array([rng.choice((0, rng.randint(0, 1 << 24), rng.randint(0, 1 << 33)))
                  for _ in range(n)])
    A = np.array([rng.randrange(8) for _ in range(n)])
    for mode in ("corrected", "verbatim"):
        ob = occupancy_batch(archs, np.stack([T, R, S], 1), mode, arch_index=A)
        o = oracle.occupancy_many(archs, A, T, np.minimum(R, 0xFFFF),
                                  np.minimum(S, 0xFFFFFFFF), verbatim=mode == "verbatim")
        illegal = o["status"] != 0
        np.testing.assert_array_equal(ob.raw["status"] == 2, illegal)
        ok = ~illegal
        for f_gpu, f_or in (("wpb", "wpb"), ("limit_warps", "lw"), ("limit_regs", "lr"),
                            ("limit_smem", "ls"), ("active_blocks", "blocks"),
                            ("active_warps", "aw"), ("limiter", "limiter"),
                            ("reg_warp_limit", "rwl")):
            np.testing.assert_array_equal(ob.raw[f_gpu][ok].astype(np.int64), o[f_or][ok],
                                          err_msg=f"{f_gpu} seed {seed} {mode}")
        np.testing.assert_array_equal(ob.raw["occupancy"][ok].view(np.int64),
                                      o["occ"][ok].view(np.int64))


@pytest.mark.parametrize("seed", range(4))
def test_random_suggest_vs_oracle(seed):
    import paper_1701_08547_b200 as P
    from paper_1701_08547_b200.batch import suggest_batch
    rng = random.Random(99 + seed)
    archs = [random_arch(rng, i) for i in range(6)]
    reqs, want = [], []
    for _ in range(3000):
        a = rng.choice(archs)
        regs = rng.choice((0, rng.randint(0, a.max_regs_per_thread), a.max_regs_per_thread))
        smem = rng.choice((0, rng.randint(0, a.shared_mem_per_block), a.shared_mem_per_block))
        if not pyref.thread_candidates(a):
            continue
        reqs.append((a, P.KernelResources("k", regs, smem)))
        want.append(pyref.suggest(a, regs, smem))
    for mode in ("corrected", "verbatim"):
        if mode == "verbatim":
            want = [pyref.suggest(a, r.registers_per_thread, r.static_shared_mem, True)
                    for a, r in reqs]
        got = suggest_batch(reqs, mode)
        for g, w in zip(got, want):
            assert (g.thread_candidates, g.register_headroom, g.smem_budget, g.best_occupancy,
                    g.best_threads, g.best_blocks) == \
                (w["thread_candidates"], w["register_headroom"], w["smem_budget"],
                 w["best_occupancy"], w["best_threads"], w["best_blocks"])


def test_random_mixes_features_vs_pyref():
    from paper_1701_08547_b200.batch import feature_score
    rng = random.Random(4242)
    mixes = [random_mix(rng) for _ in range(2000)]
    ccs = [2.0, 3.5, 5.2, 6.0, 6.1, 9.0]
    for scale in (1.0, 0.1, 3.0):
        fb = feature_score(mixes, ccs, scale=scale)
        for m, mix in enumerate(mixes):
            counts = {c.value: n for c, n in mix.counts.items()}
            assert fb.intensity[m] == pyref.intensity(counts) or \
                (np.isnan(fb.intensity[m]) and np.isnan(pyref.intensity(counts)))
            for j, cc in enumerate(ccs):
                try:
                    want = pyref.cost_estimate(counts, mix.reg_operands, cc, scale)
                except pyref.OracleUnsupported:
                    with pytest.raises(Exception):
                        fb.one(m, j)
                    continue
                got = fb.one(m, j)
                assert got.cost.hex() == want.hex()
                assert [x.hex() for x in got.shares.values()] == \
                    [x.hex() for x in pyref.pipeline_utilization(counts, mix.reg_operands,
                                                                 cc).values()]


def _k0_run(rec_dev, off, lut):
    import torch
    from paper_1701_08547_b200 import _lib, batch
    n = len(off) - 1
    d = batch.mix_reduce(rec_dev, batch._to_device(off), n, batch._to_device(lut), len(lut))
    torch.cuda.synchronize()
    return batch._to_host(d, _lib.MIX, n)


def _k0_check(out, rec, off, lut):
    counts, order, regs = oracle.aggregate_records(rec, off, lut)
    np.testing.assert_array_equal(out["counts"][:, :15].astype(np.int64), counts)
    np.testing.assert_array_equal(out["reg_operands"].astype(np.int64), regs)
    np.testing.assert_array_equal(out["n_instr"].astype(np.int64), np.diff(off.astype(np.int64)))
    fk = np.where(out["counts"][:, :15] > 0, out["first_key"][:, :15].astype(np.int64), 1 << 40)
    got = np.argsort(fk, axis=1, kind="stable")
    mask = np.arange(15)[None, :] < (counts > 0).sum(1)[:, None]
    np.testing.assert_array_equal(np.where(mask, got, -1), order)


@pytest.mark.parametrize("seed", range(6))
def test_k0_ragged_segments_vs_oracle(seed):
    """K0 on ragged CSR layouts: empty kernels (leading, interior, trailing),
    1-record kernels, kernels longer than a warp's record share, a nonzero
    first offset, and record buffers at every 4-byte misalignment (the
    vector path needs 16-byte alignment; the scalar path covers the rest)."""
    import torch
    from paper_1701_08547_b200 import batch
    rng = np.random.default_rng(1000 + seed)
    n_sig = int(rng.integers(1, 3000))
    lut = rng.integers(0, 15, n_sig).astype(np.uint8)
    kind = seed % 3
    n_k = int(rng.integers(1, 5000))
    if kind == 0:       # mostly tiny, many empty
        lens = rng.integers(0, 40, n_k) * (rng.random(n_k) > 0.3)
    elif kind == 1:     # a few huge kernels among normal ones
        lens = rng.integers(32, 2048, n_k)
        lens[rng.integers(0, n_k, 3)] = rng.integers(200_000, 2_000_000, 3)
    else:               # empties at both ends
        lens = rng.integers(1, 3000, n_k)
        lens[:5] = 0
        lens[-7:] = 0
    n_rec = int(lens.sum())
    lead = int(rng.integers(0, 9))          # records before the first kernel
    sig = rng.integers(0, n_sig, n_rec + lead).astype(np.uint32)
    regops = rng.integers(0, 256, n_rec + lead).astype(np.uint32)
    guard = (rng.random(n_rec + lead) < 0.15).astype(np.uint32)
    rec = guard | (sig << 1) | (regops << 17)
    off = (lead + np.concatenate([[0], np.cumsum(lens)])).astype(np.uint64)
    for mis in (0, 1, 2, 3):
        buf = np.zeros(len(rec) + 4, np.uint32)
        buf[mis:mis + len(rec)] = rec
        d = batch._to_device(buf)
        view = d[4 * mis:]                 # byte view shifted by 4*mis bytes
        out = _k0_run(view, off, lut)
        _k0_check(out, rec, off, lut)


@pytest.mark.parametrize("table", ["identity", "permuted", "random"])
@pytest.mark.parametrize("kind", range(3))
def test_k0_fifteen_entry_tables_vs_oracle(table, kind):
    """15-entry class tables: the identity (class records, what the
    tokenizer emits -- K0 indexes its increment table by the record's low
    byte) and two 15-entry tables that are not the identity (the same
    kernel instance, generic lookup path).  Ids 15..31 are past the table
    (Unclassified); ragged layouts as above, misaligned buffers."""
    from paper_1701_08547_b200 import batch
    rng = np.random.default_rng(77 + 10 * kind + len(table))
    lut = {"identity": np.arange(15), "permuted": rng.permutation(15),
           "random": rng.integers(0, 15, 15)}[table].astype(np.uint8)
    if table == "identity":
        np.testing.assert_array_equal(lut, batch.CLASS_LUT)
    n_k = int(rng.integers(1, 4000))
    if kind == 0:
        lens = rng.integers(0, 300, n_k) * (rng.random(n_k) > 0.2)
    elif kind == 1:
        lens = rng.integers(32, 2048, n_k)
        lens[rng.integers(0, n_k, 2)] = rng.integers(100_000, 900_000, 2)
    else:
        lens = rng.integers(1, 5000, n_k)
        lens[:3] = 0
        lens[-4:] = 0
    n_rec = int(lens.sum())
    lead = int(rng.integers(0, 9))
    # mostly common classes, a few rare ones (late first occurrences)
    p = np.r_[np.full(15, 1.0), np.full(17, 0.02)]
    p[rng.integers(0, 15, 4)] = 0.001
    sig = rng.choice(32, n_rec + lead, p=p / p.sum()).astype(np.uint32)
    regops = rng.integers(0, 256, n_rec + lead).astype(np.uint32)
    guard = (rng.random(n_rec + lead) < 0.2).astype(np.uint32)
    rec = guard | (sig << 1) | (regops << 17)
    off = (lead + np.concatenate([[0], np.cumsum(lens)])).astype(np.uint64)
    for mis in (0, 3):
        buf = np.zeros(len(rec) + 4, np.uint32)
        buf[mis:mis + len(rec)] = rec
        d = batch._to_device(buf)
        out = _k0_run(d[4 * mis:], off, lut)
        _k0_check(out, rec, off, lut)


def random_big_block_config(rng, n_arch=3, n_kern=2):
    """Spaces whose (REGS x SMEM) blocks span many 128-candidate slices, so
    K2i's separable-table path runs; block sizes are not multiples of 128
    (slices straddle blocks and segments)."""
    from paper_1701_08547_b200 import workloads
    from paper_1701_08547_b200.batch import KernelSpec
    from paper_1701_08547_b200.tuning import TuningSpace
    archs = tuple(random_arch(rng, i) for i in range(n_arch))
    kernels = []
    for kk in range(n_kern):
        tc = tuple(sorted(rng.sample(range(32, 2049, 32), rng.randint(1, 5))))
        regs = tuple(rng.sample(range(0, 1100), rng.randint(20, 300)))
        smem = tuple(rng.choice((0, 1, 1024, 6145, 49152, 232448, rng.randint(0, 1 << 25)))
                     for _ in range(rng.randint(1, 70)))
        space = TuningSpace(tc, tuple(rng.sample(range(1, 300), rng.randint(1, 2))),
                            tuple(range(1, rng.randint(2, 3))), (16,),
                            ("", "-use_fast_math")[:rng.randint(1, 2)],
                            extra=(("REGS", regs), ("SMEM", smem)))
        n_var = len(space.unroll_factors) * len(space.compiler_flags)
        kernels.append(KernelSpec(f"k{kk}", space, tuple(random_mix(rng) for _ in range(n_var))))
    return workloads.Config("random-big", tuple(kernels), archs, rng.choice((1, 5, 16, 32)))


@pytest.mark.parametrize("seed", range(8))
def test_random_big_blocks_k2i_vs_oracle(seed):
    """K2i separable block tables (limit_by_registers over REGS, limit_by_smem
    over SMEM, min per candidate) == the C oracle and the record path, both
    modes, including key offsets (weak-scaling copies) and odd windows."""
    import paper_1701_08547_b200 as P
    rng = random.Random(5000 + seed)
    cfg = random_big_block_config(rng, n_arch=rng.randint(1, 4), n_kern=rng.randint(1, 3))
    for mode in ("corrected", "verbatim"):
        prob = oracle.problem_of(cfg, verbatim=mode == "verbatim")
        want = oracle.score_spaces(prob, oracle.spaces_of(cfg), threads=8)
        plan = P.ScorePlan(cfg.kernels, cfg.archs, mode, k=cfg.k)
        got_i = plan.score_implicit().cpu().numpy().view(np.uint64)
        assert np.array_equal(got_i, want), (seed, mode, "implicit")
        got_f = plan.score_implicit(prune=False).cpu().numpy().view(np.uint64)
        assert np.array_equal(got_f, want), (seed, mode, "implicit, no pruning")
        rec = plan.generate()
        for b, n in ((0, plan.total), (rng.randrange(plan.total), None)):
            n = plan.total - b if n is None else n
            off = rng.choice((0, 1, 3, plan.total, 7 * plan.total + 5))
            a = plan.score_implicit(b, n, key_offset=off).cpu().numpy()
            r = plan.score(plan.generate(b, n), n, index_base=b + off).cpu().numpy()
            assert np.array_equal(a, r), (seed, mode, b, n, off)
        del rec


@pytest.mark.parametrize("n_sig", [32_767, 40_000, 65_535])
def test_k0_large_signature_tables(n_sig):
    """Class tables above 64 KB switch K0 to its shallow ring (2 chunks in
    flight); the 65,535-signature maximum of the record format included."""
    import torch  # noqa: F401
    rng = np.random.default_rng(n_sig)
    lut = rng.integers(0, 15, n_sig).astype(np.uint8)
    lens = rng.integers(0, 3000, 400)
    lens[::37] = 0
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    n = int(off[-1])
    sig = rng.integers(0, n_sig, n).astype(np.uint32)
    rec = ((rng.random(n) < 0.15).astype(np.uint32) | (sig << 1) |
           (rng.integers(0, 256, n).astype(np.uint32) << 17))
    from paper_1701_08547_b200 import batch
    out = _k0_run(batch._to_device(rec), off, lut)
    _k0_check(out, rec, off, lut)


@pytest.mark.parametrize("k", [1, 32])
def test_k2_k2i_extreme_k(k):
    import paper_1701_08547_b200 as P
    rng = random.Random(77 + k)
    cfg = random_big_block_config(rng, n_arch=2, n_kern=2)
    cfg = type(cfg)(cfg.name, cfg.kernels, cfg.archs, k)
    prob = oracle.problem_of(cfg)
    want = oracle.score_spaces(prob, oracle.spaces_of(cfg), threads=4)
    plan = P.ScorePlan(cfg.kernels, cfg.archs, k=k)
    assert np.array_equal(plan.score(plan.generate(), plan.total).cpu().numpy().view(np.uint64), want)
    assert np.array_equal(plan.score_implicit().cpu().numpy().view(np.uint64), want)
